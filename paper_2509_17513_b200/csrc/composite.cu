// Front-to-back alpha compositing over 16x16 tiles (render.py:301-356),
// resumable across depth-rank rounds.
//
// A round hands every tile the records of its splats whose depth ranks fall
// in the round's range, in rank order.  Running the rounds in order is the
// reference's per-pixel loop (render.py:307-332): integer rect clip,
// T < 1e-4 skip, power clamp, 0.99 alpha cap, alpha <= 0 skip, fp32
// accumulation in a fixed order (deterministic).  The first round starts
// from (C, T) = (0, 1) in registers; a tile whose pixels all saturate is
// finished on the spot (background blend, clip, u8 rounding: render.py:
// 333-338, 356, 165-169) and marked done so later rounds emit no keys for
// it; the others carry their (C, T) to the next round through `state`, and
// the last round finishes every tile still open.
#include <stdint.h>

#include <type_traits>
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

// Same with the whole warp: 32 probes per step (about log32(n) dependent
// loads instead of log2(n)); every lane returns the result.
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* __restrict__ k, uint32_t n, uint32_t t) {
    const int lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + (uint32_t)lane * step;
        const bool lt = p < hi && __ldg(k + p) < t;
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, lt));  // probes below t
        if (c == 0) return lo;
        const uint32_t nlo = lo + (c - 1) * step + 1;
        hi = min(hi, lo + c * step);
        lo = nlo;
    }
    const uint32_t p = lo + (uint32_t)lane;
    const bool lt = p < hi && __ldg(k + p) < t;
    return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// Packed fp32 pair arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a): the
// compositor's per-pixel fp32 work runs on row pairs, halving its FMA-pipe
// issue.  Rounding is the scalar ops' (.rn), so results are bit-identical to
// evaluating the pair one row at a time.
struct f2 {
    float x, y;
};
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// Upper bound of the power of one pixel: 0 when the pixel composites this
// splat (bit `bit` of m set: inside the rect; and T >= 1e-4, render.py:
// 316-318), -inf otherwise (alpha 0: C and T unchanged).
__device__ __forceinline__ float pix_lim(uint32_t m, uint32_t bit, float T) {
    float r;
    asm("{\n\t.reg .pred pm, pt;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.b32 pm, t, 0;\n\t"
        "setp.ge.and.f32 pt, %3, 0f38D1B717, pm;\n\t"
        "selp.f32 %0, 0f00000000, 0fFF800000, pt;\n\t}"
        : "=f"(r) : "r"(m), "r"(bit), "f"(T));
    return r;
}
// T if the pixel takes this splat (rect bit set and T >= 1e-4), else 0: a
// zero weight leaves C and T unchanged, exactly like the reference's skip
__device__ __forceinline__ float t_eff(uint32_t m, uint32_t bit, float T) {
    float r;
    asm("{\n\t.reg .pred pm, pt;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.b32 pm, t, 0;\n\t"
        "setp.ge.and.f32 pt, %3, 0f38D1B717, pm;\n\t"
        "selp.f32 %0, %3, 0f00000000, pt;\n\t}"
        : "=f"(r) : "r"(m), "r"(bit), "f"(T));
    return r;
}
// T if T >= 1e-4, else 0 (the rect test done by the caller)
__device__ __forceinline__ float t_live(float T) {
    float r;
    asm("{\n\t.reg .pred pt;\n\tsetp.ge.f32 pt, %1, 0f38D1B717;\n\tselp.f32 %0, %1, 0f00000000, pt;\n\t}"
        : "=f"(r) : "f"(T));
    return r;
}
__device__ __forceinline__ void sts_f4(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}
__device__ __forceinline__ float ex2f(float x) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
    return e;
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
//
// V3 (the default): the staging lane also rewrites the record's first 16 B as
// (bx, by, mask, log2 op), so a lane's per-record work is three shared loads
// (that quad, (ca, cb), (cc, r, g, b)), its rows of the rect from one byte
// permute and one column-bit test against lane constants, and the 0.99 cap
// decision from log2 op; the arithmetic is V2's, op for op (only records
// with op in (0.98994, 0.99] also take the 0.99 cap, which can only round an
// alpha of 0.99 + 1 ulp down to the reference's ceiling).
//
// V4 (CT = true, default): the staging lane also tabulates its record's
// per-column terms for the 16 columns of the tile -- A_c = dx (ca dx) +
// log2 op (-inf outside the rect's columns) and B_c = cb dx with dx = c + bx
// -- and the dy pairs of the two lane halves, so a lane's per-record work is
// loads: (A, B) of its column, its half's dy pair, (cc, r, g, b), and the
// mask / log2-op pair.  The arithmetic is V3's, op for op (bit-identical).
// The table rows are 17 float2 apart (bank-conflict-free both ways).
//
// FLAG0: every strip reads the tile's state from strip 0's flag byte (a last
// round split finer than round 1, whose ROWS = 8 warps set only strip 0).
//
// DYT (V5, with CT): the table row also holds both lane halves' four
// (dy, dy + 1) pairs (rows 208 B apart), so no lane adds the row offsets.
template <int ROWS, bool PACKED, bool TEFF, bool RANGES, bool V3 = false, int MINB = 5, int WPC = 4,
          bool CT = false, bool FLAG0 = false, bool DYT = false>
__global__ void __launch_bounds__(32 * WPC) __maxnreg__(WPC == 6 ? 112 : MINB >= 9 ? 64 : MINB >= 8 ? 72 : MINB >= 7 ? 80 : MINB >= 6 ? 88 : MINB >= 5 ? 96 : 128) composite_strip_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ tile_off, const uint32_t* __restrict__ ranks,
    const unsigned long long* __restrict__ nkeys, const SplatRec* __restrict__ recs,
    float4* __restrict__ state, uint8_t* __restrict__ tile_done, int width, int height, int ntx,
    int ntiles, bool first, bool last, float bg0, float bg1, float bg2, float* __restrict__ out_rgb,
    uint8_t* __restrict__ out_rgb8) {
    constexpr int kStrips = 16 / (2 * ROWS);  // warps per tile, each fully independent
    __shared__ __align__(16) float4 s_rec[2][WPC][32 * 4];  // double-buffered per-warp batches
    constexpr int kRow = DYT ? 26 : 17;  // float2 per table row
    __shared__ __align__(16) float2 s_ct[CT ? WPC : 1][CT ? 32 * kRow : 1];  // V4 column tables
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * WPC + warp;
    const int tile = gw / kStrips, strip = gw % kStrips;
    if (tile >= ntiles) return;
    // per-strip state: saturated strips were written out in an earlier round;
    // blank ones too, unless this round brings their tile keys
    uint8_t* flag = tile_done + 4 * (size_t)tile + (FLAG0 ? 0 : strip);
    const uint8_t td = first ? kTileOpen : *flag;
    if (td == kTileSaturated) return;
    const uint32_t K = (uint32_t)*nkeys;
    // tile range: from the round-1 binning's offsets, or a search of the
    // sorted tile keys
    uint32_t start, end;
    if constexpr (RANGES) {
        start = min(__ldg(tile_off + tile), K);
        end = min(__ldg(tile_off + tile + 1), K);
    } else {
        start = warp_lower_bound(keys, K, (uint32_t)tile);
        end = warp_lower_bound(keys, K, (uint32_t)tile + 1);
    }
    bool on = true;
    const int tx = on ? tile % ntx : 0, ty = on ? tile / ntx : 0;
    const int px = tx * kTile + (lane & 15);
    const int sy0 = ty * kTile + strip * 2 * ROWS;  // strip's first row
    const int py0 = sy0 + (lane >> 4) * ROWS;        // this lane's first row
    // lane constants against the staged per-(record, tile) fields below
    const float colf = (float)(lane & 15);                          // column in the tile
    const int rowoff = strip * 2 * ROWS + (lane >> 4) * ROWS;       // first row in the tile
    const float rowf = (float)rowoff;
    const uint32_t colsh = (uint32_t)(lane & 15), rowsh = 16u + (uint32_t)rowoff;
    // V3: the lane's column bit and the byte permute that moves its 8 rows of
    // the rect's row mask (mask bits 16-31) to bits 0-7
    const uint32_t colbit = 1u << colsh, rsel = 0x4440u | (rowsh >> 3);
    // V4: this lane's entry of record 0 in the warp's column table, and the
    // offset of its half's dy pair in a staged record
    const uint32_t ct_lane = CT ? (uint32_t)__cvta_generic_to_shared(&s_ct[warp][0]) + 8u * colsh : 0u;
    const uint32_t dy_off = 16u + 8u * (uint32_t)(lane >> 4);
    const uint32_t ct_row0 = CT ? (uint32_t)__cvta_generic_to_shared(&s_ct[warp][0]) + 128u + 32u * (uint32_t)(lane >> 4)
                                : 0u;
    float T[ROWS], c0[ROWS], c1[ROWS], c2[ROWS];
    uint32_t live = 0, inimg = 0;
    const bool work = on && start < end;
    if (td == kTileBlank && !work) on = false;  // still background, already written
    // state I/O: the first round and blank tiles start from (0, 1); open tiles
    // load it when they have keys or must be finished
    const bool load = on && !first && td == kTileOpen && (work || last);
#pragma unroll
    for (int j = 0; j < ROWS; j++) {
        T[j] = 1.f;
        c0[j] = c1[j] = c2[j] = 0.f;
        if (on && px < width && py0 + j < height) {
            inimg |= 1u << j;
            if (load) {
                const float4 st = state[(size_t)(py0 + j) * width + px];
                c0[j] = st.x;
                c1[j] = st.y;
                c2[j] = st.z;
                T[j] = st.w;
            }
            if (T[j] >= 1e-4f) live |= 1u << j;
        }
    }
    // records arrive by cp.async one batch (32 records) ahead, double
    // buffered per warp; the rank of the batch after that is loaded a batch
    // ahead too, so neither the rank nor the record gather sits in front of
    // the compositing (round 2's few open tiles are latency-bound)
    // the warp's two batch buffers (arithmetic, not an indexed local array)
    const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(&s_rec[0][warp][0]);
    constexpr uint32_t kBufStride = (uint32_t)(sizeof(float4) * WPC * 32 * 4);
    auto sb = [&](int i) { return sb0 + (uint32_t)(i & 1) * kBufStride; };
    auto issue = [&](uint32_t dst, uint32_t jr, uint32_t rank) {
        if (jr < end) {
            const char* src = reinterpret_cast<const char*>(recs + rank);
#pragma unroll
            for (int k = 0; k < 4; k++)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + lane * 64u + 16u * k),
                             "l"(src + 16 * k));
        }
        asm volatile("cp.async.commit_group;");
    };
    uint32_t rank_nx = 0;
    if (work) {
        issue(sb(0), start + lane, start + lane < end ? __ldg(ranks + start + lane) : 0u);
        rank_nx = start + 32 + lane < end ? __ldg(ranks + start + 32 + lane) : 0u;
    }
    int it = 0;
    for (uint32_t base = start; work && base < end; base += 32, it++) {
        if (!__any_sync(0xffffffffu, live)) break;
        const uint32_t sbase = sb(it);
        const bool more = base + 32 < end;
        if (more) {
            issue(sb(it + 1), base + 32 + lane, rank_nx);
            rank_nx = base + 64 + lane < end ? __ldg(ranks + base + 64 + lane) : 0u;
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        if (base + lane < end) {
            // tile-relative fields once per (record, tile) instead of per lane
            // and record: slot 0 = (bx, by, mask) with dx = column + bx, dy =
            // row + by, mask = the rect's columns (bits 0-15) and rows (bits
            // 16-31) in this tile
            const uint32_t sl = sbase + lane * 64u;
            const float4 v0 = lds_f4(sl), v1 = lds_f4(sl + 16u), v3 = lds_f4(sl + 48u);
            const uint32_t rx = __float_as_uint(v3.y), ry = __float_as_uint(v3.z);
            const int tx0 = tx * kTile, ty0 = ty * kTile;
            const int cl = min(max((int)(rx & 0xFFFFu) - tx0, 0), 16), ch = min(max((int)(rx >> 16) - tx0, 0), 16);
            const int rl = min(max((int)(ry & 0xFFFFu) - ty0, 0), 16), rh = min(max((int)(ry >> 16) - ty0, 0), 16);
            const uint32_t cm = (0xFFFFu << cl) & ~(0xFFFFu << ch) & 0xFFFFu;
            const uint32_t rm = (0xFFFFu << rl) & ~(0xFFFFu << rh) & 0xFFFFu;
            const float bxv = ((float)tx0 - v0.x) - v1.x, byv = ((float)ty0 - v0.y) - v1.y;
            sts_f4(sl, make_float4(bxv, byv, __uint_as_float(cm | (rm << 16)), V3 ? v3.w : 0.f));
            if constexpr (CT) {
                // the per-lane V3 terms, for every column: dx = c + bx, A = dx (ca dx)
                // + log2 op (one rounding: the FFMA V3 compiles to), B = cb dx
                const float ca = v1.z, cb = v1.w, lop = v3.w;
                const uint32_t row = (uint32_t)__cvta_generic_to_shared(&s_ct[warp][lane * kRow]);
#pragma unroll
                for (int c = 0; c < 16; c++) {
                    const float dx = __fadd_rn((float)c, bxv);
                    const float A1 = ((cm >> c) & 1u) ? __fmaf_rn(dx, __fmul_rn(ca, dx), lop) : -INFINITY;
                    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(row + 8u * c), "f"(A1),
                                 "f"(__fmul_rn(cb, dx)));
                }
                // dy pairs (dy0, dy0 + 1) of the two lane halves (rows 0 and 8)
                const float d0 = __fadd_rn(0.f, byv), d8 = __fadd_rn(8.f, byv);
                sts_f4(sl + 16u, make_float4(__fadd_rn(d0, 0.f), __fadd_rn(d0, 1.f), __fadd_rn(d8, 0.f),
                                             __fadd_rn(d8, 1.f)));
                if constexpr (DYT) {  // pair j of half h: ((d + 0) + j, (d + 1) + j), as V3 adds it
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const float d = h ? d8 : d0, e0 = __fadd_rn(d, 0.f), e1 = __fadd_rn(d, 1.f);
                        sts_f4(row + 128u + 32u * h, make_float4(e0, e1, __fadd_rn(e0, 2.f), __fadd_rn(e1, 2.f)));
                        sts_f4(row + 144u + 32u * h,
                               make_float4(__fadd_rn(e0, 4.f), __fadd_rn(e1, 4.f), __fadd_rn(e0, 6.f), __fadd_rn(e1, 6.f)));
                    }
                }
            }
        }
        __syncwarp();
        const int cnt = (int)min(32u, end - base);
        for (int q = 0; q < cnt; q++) {
            const uint32_t ra = sbase + (uint32_t)q * 64u;
            const float4 rc = lds_f4(ra);  // bx, by, column | row mask of the rect in this tile[, log2 op]
            const uint32_t mw = __float_as_uint(rc.z);
            // strip rows against the rect: warp-uniform skip (a strip of 8-row
            // lanes is the whole tile: every record overlaps it)
            if (kStrips > 1 && ((mw >> (16 + strip * 2 * ROWS)) & ((1u << (2 * ROWS)) - 1u)) == 0u) continue;
            // V3: the rect covers all 16 rows of the tile (row mask 0xFFFF;
            // warp-uniform).  Such records skip the vote below: it finds
            // nothing to skip for ~97% of them, and its reduction sits on the
            // record's dependency chain
            const bool full = V3 && mw >= 0xFFFF0000u;
            // rows of the lane's column inside the rect (empty outside its columns)
            uint32_t m = 0u, need = 0xFFu;
            if (!full) {
                if constexpr (V3) {
                    m = (mw & colbit) ? __byte_perm(mw, 0u, rsel) : 0u;
                } else {
                    m = ((mw >> colsh) & 1u) ? (mw >> rowsh) & ((1u << ROWS) - 1u) : 0u;
                }
                // rows some lane still needs (rect and T >= 1e-4): one vote per
                // record, then whole row pairs no lane needs are skipped with a
                // warp-uniform branch (rect edges, saturated rows)
                need = __reduce_or_sync(0xffffffffu, m & live);
                if (!need) continue;
            }
            float4 a, r3;
            if constexpr (CT) {
                a = make_float4(0.f, 0.f, 0.f, 0.f);
                r3 = make_float4(rc.w > -0.0146f ? 1.f : 0.f, 0.f, 0.f, rc.w);
            } else if constexpr (V3) {
                float2 cab;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(cab.x), "=f"(cab.y) : "r"(ra + 24u));
                a = make_float4(0.f, 0.f, cab.x, cab.y);
                // op > 0.99 (cap path) from log2 op: log2(0.99) = -0.0144996; a
                // slightly wider test only sends a few more records through
                // the (then inactive) cap
                r3 = make_float4(rc.w > -0.0146f ? 1.f : 0.f, 0.f, 0.f, rc.w);
            } else {
                a = lds_f4(ra + 16u);  // ox, oy, ca, cb
                r3 = lds_f4(ra + 48u);  // op, rx, ry, log2 op
            }
            const float4 b = lds_f4(ra + 32u);  // cc, r, g, b
            const float op = r3.x;
            float A, B, dy0;
            f2 dyct{0.f, 0.f};
            f2 dyt[4];  // DYT: this lane half's four row-pair dy values
            if constexpr (CT) {
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(A), "=f"(B)
                             : "r"(ct_lane + (uint32_t)q * (8u * kRow)));
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(dyct.x), "=f"(dyct.y) : "r"(ra + dy_off));
                dy0 = dyct.x;
                if constexpr (DYT) {
                    const uint32_t dyrow = ct_row0 + (uint32_t)q * (8u * kRow);
                    const float4 p01 = lds_f4(dyrow), p23 = lds_f4(dyrow + 16u);
                    dyt[0] = f2{p01.x, p01.y};
                    dyt[1] = f2{p01.z, p01.w};
                    dyt[2] = f2{p23.x, p23.y};
                    dyt[3] = f2{p23.z, p23.w};
                }
            } else {
                const float dx = colf + rc.x;
                A = a.z * dx * dx;
                B = a.w * dx;
                dy0 = rowf + rc.y;
            }
            if constexpr (PACKED) {
                // row pairs; a pixel outside the rect or at T < 1e-4 gets power
                // -inf (alpha 0: C, T unchanged); opacities are >= 0 (clamped
                // in the record: a negative one draws nothing in the reference).
                // TEFF: such pixels get weight T_eff = 0 instead, and the
                // opacity is folded into the exponent (A + log2 op, from the
                // record), so alpha = 2^pw needs no multiply and, for op <=
                // 0.99, no 0.99 cap (alpha <= op); the reference's p = min(p,
                // 0) only trims rounding (the conic is positive definite)
                float A1 = (TEFF && !CT) ? A + __uint_as_float(__float_as_uint(r3.w)) : A;  // CT: tabulated
                if (V3 && !CT && !(mw & colbit)) A1 = -INFINITY;
                const f2 A2{A1, A1}, B2{B, B}, C2{b.x, b.x}, O2{op, op}, D2{dy0, dy0};
                const f2 R2{b.y, b.y}, G2{b.z, b.z}, Bl2{b.w, b.w}, M1{-1.f, -1.f};
                const f2 dy01 = CT ? dyct : add2(D2, f2{0.f, 1.f});
                auto pairs = [&](auto cap_c, auto full_c) {
                    constexpr bool CAP = decltype(cap_c)::value;
                    constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
                    for (int j = 0; j < ROWS; j += 2) {
                        // FULL: no per-pair skip (nearly every pair is needed when
                        // the rect spans the tile's rows), so the four pairs form
                        // independent chains the scheduler interleaves (ex2
                        // latency hidden within the warp); a dead pair composites
                        // with weight 0
                        if (!FULL && !(need & (3u << j))) continue;
                        // (j, j) broadcast: an immediate operand, no pair constant to build
                        const f2 dy = DYT ? dyt[j / 2] : (j ? add2(dy01, f2{(float)j, (float)j}) : dy01);
                        f2 pw = fma2(fma2(C2, dy, B2), dy, A2);
                        f2 te, al;
                        if (FULL) {
                            // every row of the tile inside the rect: only the
                            // T >= 1e-4 test per pixel; a lane outside the
                            // rect's columns has A = -inf (alpha 0)
                            te = f2{t_live(T[j]), t_live(T[j + 1])};
                            al = f2{ex2f(pw.x), ex2f(pw.y)};
                        } else if (TEFF) {
                            te = f2{t_eff(m, 1u << j, T[j]), t_eff(m, 1u << (j + 1), T[j + 1])};
                            al = f2{ex2f(pw.x), ex2f(pw.y)};
                        } else {
                            pw.x = fminf(pw.x, pix_lim(m, 1u << j, T[j]));
                            pw.y = fminf(pw.y, pix_lim(m, 1u << (j + 1), T[j + 1]));
                            te = f2{T[j], T[j + 1]};
                            al = mul2(O2, f2{ex2f(pw.x), ex2f(pw.y)});
                        }
                        if (CAP) {
                            al.x = fminf(al.x, 0.99f);
                            al.y = fminf(al.y, 0.99f);
                        }
                        const f2 w = mul2(te, al);
                        f2 c = fma2(w, R2, f2{c0[j], c0[j + 1]});
                        c0[j] = c.x;
                        c0[j + 1] = c.y;
                        c = fma2(w, G2, f2{c1[j], c1[j + 1]});
                        c1[j] = c.x;
                        c1[j + 1] = c.y;
                        c = fma2(w, Bl2, f2{c2[j], c2[j + 1]});
                        c2[j] = c.x;
                        c2[j + 1] = c.y;
                        const f2 t = fma2(w, M1, f2{T[j], T[j + 1]});  // T (1 - alpha)
                        T[j] = t.x;
                        T[j + 1] = t.y;
                    }
                };
                if (full) {
                    // the rect covers the tile's 16 rows (about 60% of the
                    // (record, tile) pairs at config 2)
                    if (op == 0.f) pairs(std::false_type{}, std::true_type{});
                    else pairs(std::true_type{}, std::true_type{});
                } else if (TEFF && (V3 ? op == 0.f : op <= 0.99f)) {
                    pairs(std::false_type{}, std::false_type{});
                } else {
                    pairs(std::true_type{}, std::false_type{});
                }
            } else {
                // branch-free over the lane's rows: a pixel outside the rect or
                // already at T < 1e-4 gets alpha 0, and alpha <= 0 composites as a
                // no-op (C, T unchanged), so the ROWS chains interleave
#pragma unroll
                for (int j = 0; j < ROWS; j++) {
                    const float dy = dy0 + (float)j;
                    const float pw = fminf(fmaf(fmaf(b.x, dy, B), dy, A), 0.0f);
                    const float al = fminf(fmaxf(op * ex2f(pw), 0.0f), 0.99f);
                    float alpha;  // row bit of m and T >= 1e-4, as one bit test + one compare
                    asm("{\n\t.reg .pred pm, pt;\n\t.reg .b32 t;\n\t"
                        "and.b32 t, %1, %2;\n\tsetp.ne.b32 pm, t, 0;\n\t"
                        "setp.ge.and.f32 pt, %3, 0f38D1B717, pm;\n\t"
                        "selp.f32 %0, %4, 0f00000000, pt;\n\t}"
                        : "=f"(alpha) : "r"(m), "r"(1u << j), "f"(T[j]), "f"(al));
                    const float w = T[j] * alpha;
                    c0[j] = fmaf(w, b.y, c0[j]);
                    c1[j] = fmaf(w, b.z, c1[j]);
                    c2[j] = fmaf(w, b.w, c2[j]);
                    T[j] = T[j] - w;  // T (1 - alpha)
                }
            }
        }
        // live pixels for the early exit and the skip test, once per batch
        live = 0;
#pragma unroll
        for (int j = 0; j < ROWS; j++) live |= (T[j] >= 1e-4f ? 1u : 0u) << j;
        live &= inimg;
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    const bool tsat = __all_sync(0xffffffffu, (live & inimg) == 0);
    if (!on) return;
    // finish the strip (background blend, clip: render.py:333-338, 356) when
    // it saturated, in the last round, and as blank background when the first
    // round brought it no key; otherwise carry (C, T) to the next round
    const bool blank = first && !work && !last;
    if (last || tsat || blank) {
#pragma unroll
        for (int j = 0; j < ROWS; j++) {
            if (!((inimg >> j) & 1u)) continue;
            const size_t pix = (size_t)(py0 + j) * width + px;
            const float v[3] = {fmaf(T[j], bg0, c0[j]), fmaf(T[j], bg1, c1[j]), fmaf(T[j], bg2, c2[j])};
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const float x = fminf(fmaxf(v[k], 0.0f), 1.0f);
                if (out_rgb) out_rgb[3 * pix + k] = x;
                // write_ppm's u8 = floor(p * 255 + 0.5) (render.py:165-169) of this
                // fp32 value, exactly: x * 255 and + 0.5 are exact in fp64
                if (out_rgb8) out_rgb8[3 * pix + k] = (uint8_t)floor(__dadd_rn(__dmul_rn((double)x, 255.0), 0.5));
            }
        }
        if (lane == 0 && !last) *flag = tsat ? kTileSaturated : kTileBlank;
    } else if (work) {
#pragma unroll
        for (int j = 0; j < ROWS; j++)
            if ((inimg >> j) & 1u)
                state[(size_t)(py0 + j) * width + px] = make_float4(c0[j], c1[j], c2[j], T[j]);
        if (lane == 0 && td != kTileOpen) *flag = kTileOpen;
    }
}

int composite_rows() {
    static int rows = 0;
    if (!rows) {
        const char* e = getenv("GSV_COMPOSITE_ROWS");
        rows = e ? atoi(e) : 8;
        if (rows != 2 && rows != 4 && rows != 8) rows = 8;
    }
    return rows;
}

void launch_composite_round(const uint32_t* keys, const uint32_t* tile_off, const uint32_t* ranks,
                            const unsigned long long* nkeys, const SplatRec* recs, float4* state,
                            uint8_t* tile_done, const CamDev& cam, bool first, bool last, float* out_rgb,
                            uint8_t* out_rgb8, cudaStream_t s) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    const int ntiles = ntx * nty;
    const int rows = composite_rows();
    const int warps = ntiles * (16 / (2 * rows));
    // (warps per CTA, CTAs per SM): (1, 28) = 28 warps at <= 72 registers
    // (V4 default), (4, 5) = 20 warps at <= 96, (4, 4) = 16 warps at <= 128,
    // (6, 3) = 18 warps at <= 112
    static int cfg = -1;
    if (cfg < 0) {
        const char* e = getenv("GSV_COMPOSITE_CFG");
        cfg = e ? atoi(e) : 0;
    }
    static int packed = -1;
    if (packed < 0) {
        const char* e = getenv("GSV_COMPOSITE_PACKED");
        packed = e ? atoi(e) : 4;
    }
#define GSV_COMPOSITE_W(R, P, E, V, MB, W) GSV_COMPOSITE_X(R, P, E, V, MB, W, false)
#define GSV_COMPOSITE_X(R, P, E, V, MB, W, CTB) GSV_COMPOSITE_Y(R, P, E, V, MB, W, CTB, false)
#define GSV_COMPOSITE_Y(R, P, E, V, MB, W, CTB, DY)                                                     \
    do {                                                                                                \
        const unsigned grid = (unsigned)((warps + (W)-1) / (W));                                        \
        if (tile_off)                                                                                   \
            composite_strip_kernel<R, P, E, true, V, MB, W, CTB, false, DY><<<grid, 32 * (W), 0, s>>>(  \
                keys, tile_off, ranks, nkeys, recs, state, tile_done, cam.width, cam.height, ntx, ntiles, first, \
                last, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_rgb8);                              \
        else                                                                                            \
            composite_strip_kernel<R, P, E, false, V, MB, W, CTB, false, DY><<<grid, 32 * (W), 0, s>>>( \
                keys, tile_off, ranks, nkeys, recs, state, tile_done, cam.width, cam.height, ntx, ntiles, first, \
                last, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_rgb8);                              \
    } while (0)
#define GSV_COMPOSITE(R, P, E, V, MB) GSV_COMPOSITE_W(R, P, E, V, MB, 4)
    static int minb = -1;  // CTAs per SM the register budget is cut for (V3)
    if (minb < 0) {
        const char* e = getenv("GSV_COMPOSITE_MINB");
        minb = e ? atoi(e) : 5;
    }
    static int r2rows = -1;  // rows per lane of a last round after a first one (GSV_R2_ROWS: 8, 4 or 2)
    if (r2rows < 0) {
        const char* e = getenv("GSV_R2_ROWS");
        r2rows = e ? atoi(e) : 8;
        if (r2rows != 2 && r2rows != 4) r2rows = 8;
    }
    if (!first && last && rows == 8 && r2rows != 8 && tile_off) {
        // the few tiles still open after round 1 walk long record lists one
        // warp each; 2 (ROWS = 4) or 4 (ROWS = 2) warps per tile shorten that
        // latency-bound walk
        const unsigned g4 = (unsigned)((ntiles * (16 / (2 * r2rows)) + 3) / 4);
        if (r2rows == 4)
            composite_strip_kernel<4, true, false, true, false, 5, 4, false, true><<<g4, 128, 0, s>>>(
                keys, tile_off, ranks, nkeys, recs, state, tile_done, cam.width, cam.height, ntx, ntiles, first,
                last, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_rgb8);
        else
            composite_strip_kernel<2, true, false, true, false, 5, 4, false, true><<<g4, 128, 0, s>>>(
                keys, tile_off, ranks, nkeys, recs, state, tile_done, cam.width, cam.height, ntx, ntiles, first,
                last, cam.bg[0], cam.bg[1], cam.bg[2], out_rgb, out_rgb8);
        return;
    }
    if (packed == 5 && rows == 8) {
        GSV_COMPOSITE_Y(8, true, true, true, 5, 4, true, true);
    } else if (packed == 4 && rows == 8) {
        // warps (tiles) per CTA (GSV_COMPOSITE_WPC, default 1): one-warp CTAs
        // free a tile's registers and shared memory the moment its warp ends,
        // instead of holding them until the slowest of the CTA's four tiles
        // ends (tiles differ a lot in record count), and cap the registers at
        // 72 (GSV_COMPOSITE_REGS: 64 / 72 / 80 / 88 / 96; none spill in the
        // one-warp form): 28 resident warps per SM; +4.7% (96 registers) and
        // +2.8% more (72) over four-warp CTAs at 96, bit-identical
        // (profiles/round2/ab_warps_per_cta.txt)
        static int wpc = -1, regs = -1;
        if (wpc < 0) {
            const char* e = getenv("GSV_COMPOSITE_WPC");
            wpc = e ? atoi(e) : 1;
            e = getenv("GSV_COMPOSITE_REGS");
            regs = e ? atoi(e) : 72;
        }
        if (wpc == 1) {
            if (regs <= 64) GSV_COMPOSITE_X(8, true, true, true, 9, 1, true);
            else if (regs <= 72) GSV_COMPOSITE_X(8, true, true, true, 8, 1, true);
            else if (regs <= 80) GSV_COMPOSITE_X(8, true, true, true, 7, 1, true);
            else if (regs <= 88) GSV_COMPOSITE_X(8, true, true, true, 6, 1, true);
            else GSV_COMPOSITE_X(8, true, true, true, 5, 1, true);
        } else if (wpc == 2) GSV_COMPOSITE_X(8, true, true, true, 5, 2, true);
        else GSV_COMPOSITE_X(8, true, true, true, 5, 4, true);
    } else if (packed == 3 && rows == 8) {
        if (cfg == 2) GSV_COMPOSITE_W(8, true, true, true, 3, 6);
        else if (minb == 4 || cfg == 1) GSV_COMPOSITE(8, true, true, true, 4);
        else GSV_COMPOSITE(8, true, true, true, 5);
    } else if (packed >= 2 && rows == 8) {
        GSV_COMPOSITE(8, true, true, false, 5);
    } else if (packed) {
        if (rows == 8) GSV_COMPOSITE(8, true, false, false, 5);
        else if (rows == 4) GSV_COMPOSITE(4, true, false, false, 5);
        else GSV_COMPOSITE(2, true, false, false, 5);
    } else {
        if (rows == 8) GSV_COMPOSITE(8, false, false, false, 5);
        else if (rows == 4) GSV_COMPOSITE(4, false, false, false, 5);
        else GSV_COMPOSITE(2, false, false, false, 5);
    }
#undef GSV_COMPOSITE
#undef GSV_COMPOSITE_W
#undef GSV_COMPOSITE_X
#undef GSV_COMPOSITE_Y
}

}  // namespace gsv
