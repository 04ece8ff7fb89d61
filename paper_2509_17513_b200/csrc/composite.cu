// Front-to-back alpha compositing over 16x16 tiles (render.py:301-356),
// resumable across depth-rank rounds.
//
// One CTA per tile, one thread per pixel.  A round hands every tile the
// records of its splats whose depth ranks fall in the round's range, in rank
// order; the pixel's (C, T) state is loaded from and stored back to
// `state`, so running the rounds in order is the same per-pixel loop as the
// reference's (render.py:307-332): integer rect clip, T < 1e-4 skip, power
// clamp, 0.99 alpha cap, alpha <= 0 skip, fp32 accumulation in a fixed
// order (deterministic).  Records are staged through shared memory 256 at a
// time; each warp skips records whose rect misses its two pixel rows, and
// the CTA stops as soon as every pixel has saturated, marking the tile done
// so later rounds emit no keys for it.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

__global__ void __launch_bounds__(256) composite_round_kernel(
    const uint32_t* __restrict__ ranks, const uint32_t* __restrict__ range,
    const SplatRec* __restrict__ recs, float4* __restrict__ state, uint8_t* __restrict__ tile_done,
    int width, int height, int ntx) {
    __shared__ float4 s_a[256], s_b[256];
    __shared__ uint4 s_c[256];
    const int tile = blockIdx.x;
    const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
    if (start >= end) return;
    const int tx = tile % ntx, ty = tile / ntx;
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const int wy0 = ty * kTile + 2 * (threadIdx.x >> 5);  // this warp's two pixel rows
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
            s_a[threadIdx.x] = __ldg(r);
            s_b[threadIdx.x] = __ldg(r + 1);
            s_c[threadIdx.x] = __ldg(reinterpret_cast<const uint4*>(r + 2));
        }
        __syncthreads();
        const int cnt = (int)min(256u, end - base);
        if (!__all_sync(0xffffffffu, done)) {
            for (int q = 0; q < cnt; q++) {
                const uint4 c = s_c[q];  // op bits, rx, ry, pad
                const int y0 = (int)(c.z & 0xFFFFu), y1 = (int)(c.z >> 16);
                if (wy0 + 1 < y0 || wy0 >= y1) continue;  // warp-uniform row test
                const int x0 = (int)(c.y & 0xFFFFu), x1 = (int)(c.y >> 16);
                if (done || px < x0 || px >= x1 || py < y0 || py >= y1) continue;
                if (T < 1e-4f) {
                    done = true;
                    continue;
                }
                const float4 a = s_a[q];  // ox, oy, ca, cb
                const float4 b = s_b[q];  // cc, r, g, b
                const float dx = (float)(px - x0) - a.x;
                const float dy = (float)(py - y0) - a.y;
                float power = -0.5f * (a.z * dx * dx + 2.0f * a.w * dx * dy + b.x * dy * dy);
                power = power > 0.0f ? 0.0f : power;
                float alpha = __uint_as_float(c.x) * __expf(power);
                alpha = alpha > 0.99f ? 0.99f : alpha;
                if (alpha <= 0.0f) continue;
                const float w = T * alpha;
                c0 += w * b.y;
                c1 += w * b.z;
                c2 += w * b.w;
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

void launch_composite_round(const uint32_t* ranks, const uint32_t* range, const SplatRec* recs,
                            float4* state, uint8_t* tile_done, const CamDev& cam, cudaStream_t s) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    composite_round_kernel<<<ntx * nty, 256, 0, s>>>(ranks, range, recs, state, tile_done, cam.width,
                                                     cam.height, ntx);
}

void launch_finalize(const float4* state, const CamDev& cam, float* out_rgb, uint8_t* out_rgb8,
                     cudaStream_t s) {
    const size_t npix = (size_t)cam.width * cam.height;
    finalize_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(state, npix, cam.bg[0], cam.bg[1],
                                                                   cam.bg[2], out_rgb, out_rgb8);
}

}  // namespace gsv
