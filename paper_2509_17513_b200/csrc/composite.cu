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
#include <stdlib.h>

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

// Warp-per-strip compositor.  A 16x16 tile is split into 16/(2*ROWS) strips
// of 16 x 2*ROWS pixels, one warp each; lane l owns column l & 15 and ROWS
// consecutive rows of the strip's upper (l < 16) or lower half.  The warp
// walks the tile's records in depth-rank order, 32 at a time staged through
// its own shared-memory slot (no CTA barrier anywhere), and per record
// evaluates its ROWS pixels with the record's loads, column test and
// row-mask amortised over them.  Per pixel the arithmetic is the reference's
// (render.py:307-332): integer-rect clip, T < 1e-4 skip (a `live` bit per
// pixel), power clamp, 0.99 alpha cap, alpha <= 0 skip, fp32, fixed order.
// The quadratic form is evaluated as A + dy (B + C dy) with A, B per
// (record, column) -- a different fp32 rounding of the same fp64 quantity.
template <int ROWS>
__global__ void __launch_bounds__(128) composite_strip_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ranks,
    const unsigned long long* __restrict__ nkeys, const SplatRec* __restrict__ recs,
    float4* __restrict__ state, uint8_t* __restrict__ tile_done, int width, int height, int ntx,
    int ntiles) {
    constexpr int kStrips = 16 / (2 * ROWS);  // warps per tile; a CTA of 4 warps holds 4/kStrips tiles
    __shared__ __align__(16) float4 s_rec[4][32 * 4];
    __shared__ int s_unsat[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 4 + warp;
    const int tile = gw / kStrips, strip = gw % kStrips;
    const bool on = tile < ntiles;
    uint32_t bound = 0;
    if (on && lane < 2) bound = lower_bound_u32(keys, (uint32_t)*nkeys, (uint32_t)tile + lane);
    const uint32_t start = __shfl_sync(0xffffffffu, bound, 0), end = __shfl_sync(0xffffffffu, bound, 1);
    const int tx = on ? tile % ntx : 0, ty = on ? tile / ntx : 0;
    const int px = tx * kTile + (lane & 15);
    const int sy0 = ty * kTile + strip * 2 * ROWS;  // strip's first row
    const int py0 = sy0 + (lane >> 4) * ROWS;        // this lane's first row
    const float pxf = (float)px, py0f = (float)py0;
    float T[ROWS], c0[ROWS], c1[ROWS], c2[ROWS];
    uint32_t live = 0;
    const bool work = on && start < end;
#pragma unroll
    for (int j = 0; j < ROWS; j++) {
        T[j] = 0.f;
        c0[j] = c1[j] = c2[j] = 0.f;
        if (work && px < width && py0 + j < height) {
            const float4 st = state[(size_t)(py0 + j) * width + px];
            c0[j] = st.x;
            c1[j] = st.y;
            c2[j] = st.z;
            T[j] = st.w;
            if (st.w >= 1e-4f) live |= 1u << j;
        }
    }
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(&s_rec[warp][0]);
    for (uint32_t base = start; work && base < end; base += 32) {
        if (!__any_sync(0xffffffffu, live)) break;
        const uint32_t jr = base + lane;
        if (jr < end) {
            const float4* r = reinterpret_cast<const float4*>(recs + __ldg(ranks + jr));
#pragma unroll
            for (int k = 0; k < 4; k++) s_rec[warp][lane * 4 + k] = __ldg(r + k);
        }
        __syncwarp();
        const int cnt = (int)min(32u, end - base);
        for (int q = 0; q < cnt; q++) {
            const uint32_t ra = sbase + (uint32_t)q * 64u;
            const float4 rc = lds_f4(ra);  // x0, y0, x1, y1 (exact integers)
            // strip rows [sy0, sy0 + 2 ROWS) against [y0, y1): warp-uniform skip
            if (rc.y >= (float)(sy0 + 2 * ROWS) || rc.w <= (float)sy0) continue;
            if (pxf < rc.x || pxf >= rc.z) continue;  // column outside the rect
            const int lo = min(max((int)rc.y - py0, 0), ROWS), hi = min(max((int)rc.w - py0, 0), ROWS);
            const uint32_t m = ((0xFFFFu << lo) & ~(0xFFFFu << hi)) & live;
            if (!m) continue;
            const float4 a = lds_f4(ra + 16u);  // ox, oy, ca, cb
            const float4 b = lds_f4(ra + 32u);  // cc, r, g, b
            const float op = lds_f4(ra + 48u).x;
            const float dx = (pxf - rc.x) - a.x;
            const float A = a.z * dx * dx, B = a.w * dx;
            const float dy0 = (py0f - rc.y) - a.y;
            // branch-free over the lane's rows (masked rows get alpha 0, which
            // leaves C and T bit-identical), so the ROWS chains interleave
            uint32_t dead = 0;
#pragma unroll
            for (int j = 0; j < ROWS; j++) {
                const float dy = dy0 + (float)j;
                const float pw = fminf(fmaf(fmaf(b.x, dy, B), dy, A), 0.0f);
                float e;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(pw));
                float alpha = fminf(op * e, 0.99f);
                alpha = ((m >> j) & 1u) && alpha > 0.0f ? alpha : 0.0f;
                const float w = T[j] * alpha;
                c0[j] = fmaf(w, b.y, c0[j]);
                c1[j] = fmaf(w, b.z, c1[j]);
                c2[j] = fmaf(w, b.w, c2[j]);
                T[j] = T[j] * (1.0f - alpha);
                dead |= (T[j] < 1e-4f ? 1u : 0u) << j;
            }
            live &= ~dead;
        }
        __syncwarp();
    }
    bool sat = true;
#pragma unroll
    for (int j = 0; j < ROWS; j++) {
        if (work && px < width && py0 + j < height) {
            state[(size_t)(py0 + j) * width + px] = make_float4(c0[j], c1[j], c2[j], T[j]);
            sat = sat && T[j] < 1e-4f;
        }
    }
    // a tile is done once all its in-image pixels are saturated; tiles this
    // round did not touch keep their flag (they were either done already or
    // receive keys in a later round)
    const bool wsat = __all_sync(0xffffffffu, sat);
    if constexpr (kStrips == 1) {
        if (work && wsat && lane == 0) tile_done[tile] = 1;
    } else {
        if (lane == 0) s_unsat[warp] = work ? (wsat ? 0 : 1) : 2;
        __syncthreads();
        if (on && strip == 0 && lane == 0) {
            bool any_work = false, all_sat = true;
            for (int k = 0; k < kStrips; k++) {
                const int u = s_unsat[warp + k];
                any_work |= u != 2;
                all_sat &= u != 1;
            }
            if (any_work && all_sat) tile_done[tile] = 1;
        }
    }
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

static int composite_rows() {
    static int rows = 0;
    if (!rows) {
        const char* e = getenv("GSV_COMPOSITE_ROWS");
        rows = e ? atoi(e) : 4;
        if (rows != 2 && rows != 4 && rows != 8) rows = 4;
    }
    return rows;
}

void launch_composite_round(const uint32_t* keys, const uint32_t* ranks,
                            const unsigned long long* nkeys, const SplatRec* recs, float4* state,
                            uint8_t* tile_done, const CamDev& cam, cudaStream_t s) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    const int ntiles = ntx * nty;
    const int rows = composite_rows();
    const int warps = ntiles * (16 / (2 * rows));
    const unsigned grid = (unsigned)((warps + 3) / 4);
    if (rows == 8)
        composite_strip_kernel<8><<<grid, 128, 0, s>>>(keys, ranks, nkeys, recs, state, tile_done, cam.width,
                                                        cam.height, ntx, ntiles);
    else if (rows == 4)
        composite_strip_kernel<4><<<grid, 128, 0, s>>>(keys, ranks, nkeys, recs, state, tile_done, cam.width,
                                                        cam.height, ntx, ntiles);
    else
        composite_strip_kernel<2><<<grid, 128, 0, s>>>(keys, ranks, nkeys, recs, state, tile_done, cam.width,
                                                        cam.height, ntx, ntiles);
}

void launch_finalize(const float4* state, const CamDev& cam, float* out_rgb, uint8_t* out_rgb8,
                     cudaStream_t s) {
    const size_t npix = (size_t)cam.width * cam.height;
    finalize_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(state, npix, cam.bg[0], cam.bg[1],
                                                                   cam.bg[2], out_rgb, out_rgb8);
}

}  // namespace gsv
