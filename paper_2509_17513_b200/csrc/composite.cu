// Front-to-back alpha compositing over 16x16 tiles (render.py:301-356).
//
// One CTA per tile, one thread per pixel.  The tile's depth-ordered splat
// records are staged through shared memory 256 at a time; every pixel walks
// them in the reference's order (global stable depth rank), applying the
// reference's per-splat integer rect clip (render.py:308-315), the
// T < 1e-4 skip (316-318), the power clamp (321-322), the 0.99 alpha cap
// (324-325) and the alpha <= 0 skip (326-327).  When every pixel of the tile
// has saturated (__syncthreads_and) the CTA stops.  Accumulation is fp32; the
// per-pixel order is fixed, so the output is deterministic.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

__global__ void __launch_bounds__(256) composite_kernel(const uint32_t* __restrict__ ranks,
                                                        const uint32_t* __restrict__ range,
                                                        const SplatRec* __restrict__ recs, int width,
                                                        int height, int ntx, float bg0, float bg1,
                                                        float bg2, float* __restrict__ out_rgb,
                                                        uint8_t* __restrict__ out_rgb8) {
    __shared__ float4 s_a[256], s_b[256];
    __shared__ uint4 s_c[256];
    const int tile = blockIdx.x;
    const int tx = tile % ntx, ty = tile / ntx;
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < width && py < height;
    const uint32_t start = range[2 * tile], end = range[2 * tile + 1];
    float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
    bool done = !inside;
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
        if (!done) {
            for (int q = 0; q < cnt; q++) {
                const uint4 c = s_c[q];  // op bits, rx, ry, pad
                const int x0 = (int)(c.y & 0xFFFFu), x1 = (int)(c.y >> 16);
                const int y0 = (int)(c.z & 0xFFFFu), y1 = (int)(c.z >> 16);
                if (px < x0 || px >= x1 || py < y0 || py >= y1) continue;
                if (T < 1e-4f) {
                    done = true;
                    break;
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
    if (!inside) return;
    const float v[3] = {c0 + T * bg0, c1 + T * bg1, c2 + T * bg2};
    const size_t o = ((size_t)py * width + px) * 3;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const float x = fminf(fmaxf(v[k], 0.0f), 1.0f);
        if (out_rgb) out_rgb[o + k] = x;
        if (out_rgb8) out_rgb8[o + k] = (uint8_t)floorf(x * 255.0f + 0.5f);
    }
}

void launch_composite(const uint32_t* ranks, const uint32_t* range, const SplatRec* recs,
                      const CamDev& cam, float* out_rgb, uint8_t* out_rgb8, cudaStream_t s) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    composite_kernel<<<ntx * nty, 256, 0, s>>>(ranks, range, recs, cam.width, cam.height, ntx,
                                               cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_rgb8);
}

}  // namespace gsv
