// Front-to-back alpha compositing over 16x16 tiles (render.py:301-356),
// resumable across depth-rank rounds.
//
// One CTA per tile, one thread per pixel, each warp an 8x4 pixel block.  A
// round hands every tile the
// records of its splats whose depth ranks fall in the round's range, in rank
// order; the pixel's (C, T) state is loaded from and stored back to
// `state`, so running the rounds in order is the same per-pixel loop as the
// reference's (render.py:307-332): integer rect clip, T < 1e-4 skip, power
// clamp, 0.99 alpha cap, alpha <= 0 skip, fp32 accumulation in a fixed
// order (deterministic).  Records are staged through shared memory 256 at a
// time; each warp ballots 32 records at a time against its block's bounds
// and walks only the hits, leaves as soon as its 32 pixels are saturated,
// and the CTA stops once every pixel has saturated, marking the tile done so
// later rounds emit no keys for it.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

// first index in the tile-sorted keys with key >= t
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ k, uint32_t n, uint32_t t) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(k + mid) < t) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

__global__ void __launch_bounds__(256) composite_round_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ranks,
    const unsigned long long* __restrict__ nkeys, const SplatRec* __restrict__ recs,
    float4* __restrict__ state, uint8_t* __restrict__ tile_done, int width, int height, int ntx) {
    __shared__ __align__(16) float4 s_rec[256 * 4];  // 256 staged 64-B records
    __shared__ uint32_t s_range[2];
    const int tile = blockIdx.x;
    if (threadIdx.x < 2) {  // this tile's [start, end) in the tile-sorted keys
        const uint32_t K = (uint32_t)*nkeys;
        s_range[threadIdx.x] = lower_bound_u32(keys, K, (uint32_t)tile + threadIdx.x);
    }
    __syncthreads();
    const uint32_t start = s_range[0], end = s_range[1];
    if (start >= end) return;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_rec);
    const int tx = tile % ntx, ty = tile / ntx;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // warp w owns an 8x4 pixel block of the 16x16 tile
    const int bx0 = tx * kTile + (warp & 1) * 8, by0 = ty * kTile + (warp >> 1) * 4;
    const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
    const float pxf = (float)px, pyf = (float)py;
    const float bx0f = (float)bx0, by0f = (float)by0;
    const bool inside = px < width && py < height;
    const size_t pix = (size_t)py * width + px;
    float4 st = inside ? state[pix] : make_float4(0.f, 0.f, 0.f, 0.f);
    float T = st.w, c0 = st.x, c1 = st.y, c2 = st.z;
    bool done = !inside || T < 1e-4f;
    for (uint32_t base = start; base < end; base += 256) {
        if (__syncthreads_and(done)) break;
        const uint32_t j = base + threadIdx.x;
        if (j < end) {
            const float4* r = reinterpret_cast<const float4*>(recs + ranks[j]);
#pragma unroll
            for (int k = 0; k < 4; k++) s_rec[threadIdx.x * 4 + k] = __ldg(r + k);
        }
        __syncthreads();
        const int cnt = (int)min(256u, end - base);
        for (int g = 0; g < cnt; g += 32) {
            if (__all_sync(0xffffffffu, done)) break;
            // which of the next 32 records touch this warp's 8x4 block?
            bool hit = false;
            if (g + lane < cnt) {
                const float4 rc = lds_f4(sbase + (uint32_t)(g + lane) * 64u);
                hit = rc.x < bx0f + 8.0f && rc.z > bx0f && rc.y < by0f + 4.0f && rc.w > by0f;
            }
            uint32_t mask = __ballot_sync(0xffffffffu, hit);
            while (mask) {
                const uint32_t q = (uint32_t)(g + __ffs(mask) - 1);
                mask &= mask - 1;
                if (done) continue;
                const uint32_t ra = sbase + q * 64u;
                const float4 rc = lds_f4(ra);  // x0, y0, x1, y1
                // outside the splat's integer rect (render.py:313-315)
                if (pxf < rc.x || pxf >= rc.z || pyf < rc.y || pyf >= rc.w) continue;
                if (T < 1e-4f) {
                    done = true;
                    continue;
                }
                const float4 a = lds_f4(ra + 16u);  // ox, oy, ca, cb
                const float4 b = lds_f4(ra + 32u);  // cc, r, g, b
                const float op = lds_f4(ra + 48u).x;
                const float dx = (pxf - rc.x) - a.x;
                const float dy = (pyf - rc.y) - a.y;
                const float pw = fminf(fmaf(fmaf(a.z, dx, a.w * dy), dx, b.x * dy * dy), 0.0f);
                float e;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(pw));
                const float alpha = fminf(op * e, 0.99f);
                if (alpha <= 0.0f) continue;
                const float w = T * alpha;
                c0 = fmaf(w, b.y, c0);
                c1 = fmaf(w, b.z, c1);
                c2 = fmaf(w, b.w, c2);
                T = T * (1.0f - alpha);
            }
        }
    }
    if (inside) state[pix] = make_float4(c0, c1, c2, T);
    const bool all_done = __syncthreads_and(!inside || T < 1e-4f);
    if (threadIdx.x == 0 && all_done) tile_done[tile] = 1;
}

__global__ void state_init_kernel(float4* __restrict__ state, uint8_t* __restrict__ tile_done,
                                  size_t npix, int ntiles) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npix) state[i] = make_float4(0.f, 0.f, 0.f, 1.f);
    if (i < (size_t)ntiles) tile_done[i] = 0;
}

// background blend + clip (render.py:333-338, 356) and optional u8 like write_ppm
__global__ void finalize_kernel(const float4* __restrict__ state, size_t npix, float bg0, float bg1,
                                float bg2, float* __restrict__ out_rgb, uint8_t* __restrict__ out_rgb8) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    const float4 s = state[i];
    const float v[3] = {s.x + s.w * bg0, s.y + s.w * bg1, s.z + s.w * bg2};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const float x = fminf(fmaxf(v[k], 0.0f), 1.0f);
        if (out_rgb) out_rgb[3 * i + k] = x;
        if (out_rgb8) out_rgb8[3 * i + k] = (uint8_t)floorf(x * 255.0f + 0.5f);
    }
}

void launch_state_init(float4* state, uint8_t* tile_done, size_t npix, int ntiles, cudaStream_t s) {
    const size_t n = npix > (size_t)ntiles ? npix : (size_t)ntiles;
    state_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(state, tile_done, npix, ntiles);
}

void launch_composite_round(const uint32_t* keys, const uint32_t* ranks,
                            const unsigned long long* nkeys, const SplatRec* recs, float4* state,
                            uint8_t* tile_done, const CamDev& cam, cudaStream_t s) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    composite_round_kernel<<<ntx * nty, 256, 0, s>>>(keys, ranks, nkeys, recs, state, tile_done,
                                                     cam.width, cam.height, ntx);
}

void launch_finalize(const float4* state, const CamDev& cam, float* out_rgb, uint8_t* out_rgb8,
                     cudaStream_t s) {
    const size_t npix = (size_t)cam.width * cam.height;
    finalize_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(state, npix, cam.bg[0], cam.bg[1],
                                                                   cam.bg[2], out_rgb, out_rgb8);
}

}  // namespace gsv
