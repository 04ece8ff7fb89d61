// GPU encoder: quantisation of one group's channels and
// the codec-1 range coder, producing byte-identical payload bodies to the
// reference encoder.
//
//   quantize_channel (quantize.py:62-106) with the f32 range cover
//   (quantize.py:62-76), flatten_to_plane (quantize.py:160-167: row-major,
//   padded with the frame's last code), plane_residuals + zigzag
//   (_rc.py:249-279,319-324), encode_bittree (_rc.py:55-118) and
//   _encode_reference_body (codec.py:137-163: per-plane RAW/RC choice with
//   the model snapshot restored for RAW planes, trailing zero trim, whole-run
//   raw fallback).
//
// Compiled with -fmad=false, and the quantisation arithmetic is spelled with
// explicit round-to-nearest intrinsics, so that
// floor((v - lo) / (hi - lo) * top + 0.5) rounds exactly like numpy.
//
// The range coder is sequential within a run (one adaptive model, temporal
// predictor), so one lane encodes one run, 32 runs of the same sample width
// per warp, one warp per CTA, probabilities lane-private in shared memory in
// the decoder's layout.  Unlike the decoder every bit is known up front, so
// the 8 node probabilities of a byte are loaded together and only the
// (low, rng) recurrence is serial.  Raw blocks (RAW planes, whole-run raw
// fallback) are copied afterwards by a cooperative kernel.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "gsv_internal.h"

namespace gsv {

// ---------------------------------------------------------------------------
// Quantisation
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ord_key(double v) {  // order-preserving
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & ~(1ull << 63)) : ~k));
}

// per channel: [0] min key, [1] max key, [2] non-finite flag
__global__ void enc_minmax_kernel(const QuantChannel* __restrict__ ch, unsigned long long* __restrict__ red) {
    const QuantChannel c = ch[blockIdx.y];
    const uint64_t total = (uint64_t)c.frames * c.n;
    unsigned long long mn = ~0ull, mx = 0ull, bad = 0ull;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double v = __ldg(c.values + (i / c.n) * c.frame_stride + (i % c.n));
        if (!isfinite(v)) bad = 1ull;
        const unsigned long long k = ord_key(v);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        bad |= __shfl_xor_sync(0xFFFFFFFFu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* r = red + 3 * blockIdx.y;
        atomicMin(r, mn);
        atomicMax(r + 1, mx);
        if (bad) atomicOr(r + 2, 1ull);
    }
}

// _f32_cover (quantize.py:62-76): the f32 range that contains [min, max]
__global__ void enc_cover_kernel(const unsigned long long* __restrict__ red, int nch, float* __restrict__ ranges) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const double vmin = ord_val(red[3 * c]);
    double vmax = ord_val(red[3 * c + 1]);
    if (vmax == vmin) vmax = __dadd_rn(vmin, 1e-6);
    float lo = __double2float_rn(vmin);
    if ((double)lo > vmin) lo = nextafterf(lo, -INFINITY);
    float hi = __double2float_rn(vmax);
    if ((double)hi < vmax) hi = nextafterf(hi, INFINITY);
    while ((double)hi <= (double)lo) hi = nextafterf(hi, INFINITY);
    ranges[2 * c] = lo;
    ranges[2 * c + 1] = hi;
}

// codes = clip(floor((v - lo) / (hi - lo) * top + 0.5), 0, top) into the
// padded plane layout; one thread per output sample
__global__ void enc_quantize_kernel(const QuantChannel* __restrict__ ch, const float* __restrict__ ranges) {
    const QuantChannel c = ch[blockIdx.y];
    const uint32_t hw = c.w * c.h;
    const uint64_t total = (uint64_t)c.frames * hw;
    const double lo = (double)ranges[2 * blockIdx.y], hi = (double)ranges[2 * blockIdx.y + 1];
    const double top = c.bits >= 32 ? 4294967295.0 : (double)((1u << c.bits) - 1u);
    const double span = __dsub_rn(hi, lo);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t f = (uint32_t)(i / hw), p = (uint32_t)(i % hw);
        const uint32_t j = p < c.n ? p : c.n - 1;
        const double v = __ldg(c.values + (uint64_t)f * c.frame_stride + j);
        double q = floor(__dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(v, lo), span), top), 0.5));
        q = q < 0.0 ? 0.0 : (q > top ? top : q);
        const uint32_t code = (uint32_t)q;
        if (c.bits == 8) c.planes[i] = (uint8_t)code;
        else if (c.bits == 16) reinterpret_cast<uint16_t*>(c.planes)[i] = (uint16_t)code;
        else reinterpret_cast<uint32_t*>(c.planes)[i] = code;
    }
}

void launch_quantize(const QuantChannel* d_ch, int nch, uint64_t max_values, uint64_t max_samples,
                     unsigned long long* d_red, float* d_ranges, cudaStream_t s) {
    if (nch <= 0) return;
    auto blocks = [](uint64_t n) {
        uint64_t b = (n + 255) / 256;
        return (unsigned)(b < 1 ? 1 : (b > 148 * 4 ? 148 * 4 : b));
    };
    enc_minmax_kernel<<<dim3(blocks(max_values), nch), 256, 0, s>>>(d_ch, d_red);
    enc_cover_kernel<<<(nch + 127) / 128, 128, 0, s>>>(d_red, nch, d_ranges);
    enc_quantize_kernel<<<dim3(blocks(max_samples), nch), 256, 0, s>>>(d_ch, d_ranges);
}

// ---------------------------------------------------------------------------
// Range coder
// ---------------------------------------------------------------------------
constexpr int kEncRPW = 32;
constexpr uint32_t kEncTree = 256u * 4u;
__host__ __device__ constexpr uint32_t enc_lane_stride(int nb) { return (uint32_t)nb * kEncTree + 16u; }

__device__ __forceinline__ uint32_t e_lds(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void e_sts(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// encoder state of one plane (_rc.py:62-68)
struct RcEncState {
    unsigned long long low;
    unsigned long long whi;  // deferred mode: bits 64..127 of the low window
    uint32_t s;              // deferred mode: renormalisation bytes not yet emitted
    uint32_t rng, cache;
    uint64_t cache_size;
    uint64_t npos;   // bytes emitted (written while < cap)
    uint64_t zrun;   // trailing zero bytes emitted
    uint64_t cap, limit;
    uint8_t* dst;
    bool overflow;
};

// a run of pending 0xFF bytes (rare: cache_size > 1), out of line
__device__ __noinline__ uint64_t emit_run(uint8_t* dst, uint64_t npos, uint64_t cap, uint64_t cnt, uint32_t b) {
    for (uint64_t i = 0; i < cnt; i++, npos++)
        if (npos < cap) dst[npos] = (uint8_t)b;
    return npos;
}

// shift_low (_rc.py:98-115), applied where `act`: predicated straight-line
// code, so that the 32 lanes of a warp (32 independent runs, renormalising
// at different decisions) do not diverge; only the rare emission of a run
// of pending 0xFF bytes branches
__device__ __forceinline__ void shift_low(RcEncState& st, bool act) {
    const bool ovf = act && (st.npos + st.cache_size > st.limit);
    st.overflow |= ovf;
    act = act && !ovf;
    const uint32_t lo32 = (uint32_t)st.low;
    const uint32_t carry = (uint32_t)(st.low >> 32);
    const bool out = act && (lo32 < 0xFF000000u || carry != 0u);
    const uint32_t b = (st.cache + carry) & 0xFFu;
    if (out && st.npos < st.cap) st.dst[st.npos] = (uint8_t)b;
    if (out && st.cache_size > 1) {
        const uint32_t bf = (0xFFu + carry) & 0xFFu;
        const uint64_t np = emit_run(st.dst, st.npos + 1, st.cap, st.cache_size - 1, bf);
        st.zrun = bf ? 0 : (b ? 0 : st.zrun + 1) + st.cache_size - 1;
        st.npos = np - 1;  // the +1 below
    } else if (out) {
        st.zrun = b ? 0 : st.zrun + 1;
    }
    st.npos += out ? 1u : 0u;
    st.cache = out ? lo32 >> 24 : st.cache;
    st.cache_size = act ? (out ? 1u : st.cache_size + 1u) : st.cache_size;
    st.low = act ? (unsigned long long)(lo32 & 0x00FFFFFFu) << 8 : st.low;
}

// shift_low with branches: a lane that does not renormalise skips it (used
// when a warp carries few runs, where divergence costs little)
__device__ __forceinline__ void shift_low_br(RcEncState& st) {
    if (st.npos + st.cache_size > st.limit) {
        st.overflow = true;
        return;
    }
    const uint32_t lo32 = (uint32_t)st.low;
    const uint32_t carry = (uint32_t)(st.low >> 32);
    if (lo32 < 0xFF000000u || carry != 0u) {
        const uint32_t b = (st.cache + carry) & 0xFFu;
        if (st.npos < st.cap) st.dst[st.npos] = (uint8_t)b;
        st.zrun = b ? 0 : st.zrun + 1;
        st.npos++;
        if (st.cache_size > 1) {
            const uint32_t bf = (0xFFu + carry) & 0xFFu;
            st.npos = emit_run(st.dst, st.npos, st.cap, st.cache_size - 1, bf);
            st.zrun = bf ? 0 : st.zrun + st.cache_size - 1;
        }
        st.cache = lo32 >> 24;
        st.cache_size = 0;
    }
    st.cache_size++;
    st.low = (unsigned long long)(lo32 & 0x00FFFFFFu) << 8;
}

// Deferred emission: renormalisation only shifts a 128-bit low window
// (whi:low) and counts the byte; every 4 decisions the pending bytes are
// pushed through shift_low's cache / 0xFF-run logic at once.  The emitted
// stream is the digit string of the same big-number sum (carries that the
// eager coder applies to its cache byte have already propagated inside the
// window), so the bytes are identical, and the decision loop has no
// branches on the renormalisation.  At most 2 bytes per decision, flushed
// every 4 decisions: the window holds 33 + 64 bits.
__device__ __forceinline__ uint64_t win_shr(const RcEncState& st, uint32_t a) {  // 32 <= a <= 96
    return a >= 64 ? (st.whi >> (a - 64)) : ((st.low >> a) | (st.whi << (64 - a)));
}
__device__ __forceinline__ void flush_deferred(RcEncState& st) {
    const uint32_t s = st.s;
    if (s == 0) return;
    uint32_t carry = (uint32_t)(win_shr(st, 32 + 8 * s) & 1u);
    for (uint32_t i = 0; i < s; i++) {
        if (st.npos + st.cache_size > st.limit) {
            st.overflow = true;
            break;
        }
        const uint32_t t = (uint32_t)(win_shr(st, 32 + 8 * (s - 1 - i)) & 0xFFu);
        if (t != 0xFFu || carry != 0u) {
            const uint32_t b = (st.cache + carry) & 0xFFu;
            if (st.npos < st.cap) st.dst[st.npos] = (uint8_t)b;
            st.zrun = b ? 0 : st.zrun + 1;
            st.npos++;
            if (st.cache_size > 1) {
                const uint32_t bf = (0xFFu + carry) & 0xFFu;
                st.npos = emit_run(st.dst, st.npos, st.cap, st.cache_size - 1, bf);
                st.zrun = bf ? 0 : st.zrun + st.cache_size - 1;
            }
            st.cache = t;
            st.cache_size = 0;
        }
        st.cache_size++;
        carry = 0;
    }
    st.low &= 0xFFFFFFFFull;
    st.whi = 0;
    st.s = 0;
}

__device__ __forceinline__ void encode_byte_deferred(uint32_t T, uint32_t byte, RcEncState& st) {
    uint32_t p[8];
#pragma unroll
    for (int k = 0; k < 8; k++) p[k] = e_lds(T + 4u * ((256u | byte) >> (8 - k)));
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t bit = (byte >> (7 - k)) & 1u;
        const uint32_t bound = (st.rng >> 12) * p[k];
        const unsigned long long add = bit ? bound : 0u;
        st.low += add;
        st.whi += st.low < add ? 1u : 0u;
        st.rng = bit ? st.rng - bound : bound;
        e_sts(T + 4u * ((256u | byte) >> (8 - k)),
              p[k] + (uint32_t)(((int32_t)(bit ? 15u : 4096u) - (int32_t)p[k]) >> 4));
        const bool r1 = st.rng < (1u << 24);
        st.rng = r1 ? st.rng << 8 : st.rng;
        st.whi = r1 ? (st.whi << 8) | (st.low >> 56) : st.whi;
        st.low = r1 ? st.low << 8 : st.low;
        st.s += r1 ? 1u : 0u;
        if (st.rng < (1u << 24)) {  // rare second byte (rng < 2^16 after the decision)
            st.rng <<= 8;
            st.whi = (st.whi << 8) | (st.low >> 56);
            st.low <<= 8;
            st.s++;
        }
        if (k == 3 || k == 7) flush_deferred(st);
    }
}

// one byte through tree T (_rc.py:76-97).  The path is known, so all 8
// node probabilities are loaded up front; the decisions are unrolled and
// only rng -> bound -> rng is serial.  MODE 1: renormalise in a branch
// (few runs per warp) or predicated (full warps).
template <int MODE>
__device__ __forceinline__ void encode_byte(uint32_t T, uint32_t byte, RcEncState& st) {
    uint32_t p[8];
#pragma unroll
    for (int k = 0; k < 8; k++) p[k] = e_lds(T + 4u * ((256u | byte) >> (8 - k)));
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t bit = (byte >> (7 - k)) & 1u;
        const uint32_t bound = (st.rng >> 12) * p[k];
        st.low += bit ? bound : 0u;
        st.rng = bit ? st.rng - bound : bound;
        e_sts(T + 4u * ((256u | byte) >> (8 - k)),
              p[k] + (uint32_t)(((int32_t)(bit ? 15u : 4096u) - (int32_t)p[k]) >> 4));
        if (MODE == 1) {
            while (st.rng < (1u << 24)) {
                shift_low_br(st);
                st.rng <<= 8;
            }
        } else {
            const bool r1 = st.rng < (1u << 24);
            shift_low(st, r1);
            st.rng = r1 ? st.rng << 8 : st.rng;
            if (st.rng < (1u << 24)) {  // rare second byte (rng < 2^16 after the decision)
                shift_low(st, true);
                st.rng <<= 8;
            }
        }
    }
}

template <int NB>
__device__ __forceinline__ uint32_t ld_sample(const uint8_t* plane, uint32_t i) {
    if (NB == 1) return __ldg(plane + i);
    if (NB == 2) return __ldg(reinterpret_cast<const uint16_t*>(plane) + i);
    return __ldg(reinterpret_cast<const uint32_t*>(plane) + i);
}

template <int NB, int MODE>
__device__ void encode_run(const EncRun& r, uint32_t P, EncResult* res) {
    for (int b = 0; b < NB; b++)  // new_bittree_probs (_rc.py:304-317)
        for (uint32_t i = 0; i < 256; i++)
            e_sts(P + b * kEncTree + 4u * i, (i != 0 && (i & (i - 1)) == 0) ? 3686u : 2048u);
    const uint32_t hw = r.w * r.h, w = r.w;
    const uint64_t raw_plane = (uint64_t)hw * NB, raw_len = raw_plane * r.count;
    const uint64_t limit = raw_plane * 10 + 64 - 8;  // bittree_worst_case - 8 (_rc.py:45-47,66)
    const uint32_t mask = NB == 4 ? 0xFFFFFFFFu : (1u << (8 * NB)) - 1u, half = 1u << (8 * NB - 1);
    const uint32_t def = 128u << (8 * NB - 8);
    uint64_t wpos = 1 + (uint64_t)r.count;
    bool whole_raw = false;
    for (uint32_t f = 0; f < r.count; f++) {
        for (uint32_t i = 0; i < NB * 256u; i++) r.snap[i] = e_lds(P + 4u * i);
        const uint8_t* plane = r.samples + f * raw_plane;
        const uint8_t* prev = f > 0 ? plane - raw_plane : plane;
        RcEncState st;
        st.low = 0;
        st.whi = 0;
        st.s = 0;
        st.rng = 0xFFFFFFFFu;
        st.cache = 0;
        st.cache_size = 1;
        st.npos = 0;
        st.zrun = 0;
        st.dst = r.body + wpos + 4;
        st.cap = raw_plane;
        st.limit = limit;
        st.overflow = false;
        uint32_t x = 0, y = 0;
        // sample and predictor of the next position loaded one sample ahead
        auto predictor = [&](uint32_t i, uint32_t xx, uint32_t yy) -> uint32_t {
            if (f > 0) return ld_sample<NB>(prev, i);
            if (xx > 0) return ld_sample<NB>(plane, i - 1);
            if (yy > 0) return ld_sample<NB>(plane, i - w);
            return def;
        };
        uint32_t vn = ld_sample<NB>(plane, 0), pdn = predictor(0, 0, 0);
        for (uint32_t i = 0; i < hw && !st.overflow; i++) {
            const uint32_t v = vn, pred = pdn;
            if (i + 1 < hw) {
                const uint32_t x1 = x + 1 == w ? 0 : x + 1, y1 = x + 1 == w ? y + 1 : y;
                vn = ld_sample<NB>(plane, i + 1);
                pdn = predictor(i + 1, x1, y1);
            }
            // residual wrapped into [-half, half) (_rc.py:273-274), zigzagged
            // (_rc.py:319-324): d = (v - pred) mod 2^bits; z = 2d below half,
            // else 2 (2^bits - d) - 1
            const uint32_t d = (v - pred) & mask;
            const uint32_t z = d < half ? 2u * d : 2u * ((0u - d) & mask) - 1u;
#pragma unroll 1
            for (int b = 0; b < NB; b++) {
                if (MODE == 2) encode_byte_deferred(P + b * kEncTree, (z >> (8 * b)) & 0xFFu, st);
                else encode_byte<MODE>(P + b * kEncTree, (z >> (8 * b)) & 0xFFu, st);
            }
            if (++x == w) {
                x = 0;
                y++;
            }
        }
        if (MODE == 2) flush_deferred(st);
        for (int i = 0; i < 5; i++) shift_low(st, !st.overflow);
        const int64_t n = st.overflow ? -1 : (int64_t)(st.npos - st.zrun);
        if (n < 0 || (uint64_t)n + 4 >= raw_plane) {
            for (uint32_t i = 0; i < NB * 256u; i++) e_sts(P + 4u * i, r.snap[i]);  // probs = snapshot
            r.body[1 + f] = 1;
            r.blk_off[f] = wpos;
            wpos += raw_plane;
        } else {
            r.body[1 + f] = 0;
            uint8_t* q = r.body + wpos;
            q[0] = (uint8_t)n;
            q[1] = (uint8_t)(n >> 8);
            q[2] = (uint8_t)(n >> 16);
            q[3] = (uint8_t)(n >> 24);
            r.blk_off[f] = wpos;
            wpos += 4 + (uint64_t)n;
        }
        if (wpos > raw_len + 1) {  // the body can only grow: whole-run raw
            whole_raw = true;
            break;
        }
    }
    res->whole_raw = whole_raw ? 1u : 0u;
    res->body_len = whole_raw ? raw_len + 1 : wpos;
}

// runs per warp (c.lanes) adapts to the run count: few runs -> one run per
// warp (no divergence, branchy renormalisation), many runs -> full warps
// (predicated renormalisation)
template <int MODE>
__global__ void __launch_bounds__(kEncRPW) rc_encode_kernel(const EncRun* __restrict__ runs,
                                                            const uint32_t* __restrict__ order, EncClasses c,
                                                            EncResult* __restrict__ res) {
    extern __shared__ uint4 eprobs_s[];
    if ((int)threadIdx.x >= c.lanes) return;
    const int b = blockIdx.x;
    const int cls = b < c.blk[1] ? 0 : (b < c.blk[2] ? 1 : 2);
    const int nb = 1 << cls;
    const int gi = (b - c.blk[cls]) * c.lanes + threadIdx.x;
    if (gi >= c.n[cls]) return;
    const uint32_t ri = order[c.off[cls] + gi];
    const uint32_t P = (uint32_t)__cvta_generic_to_shared(eprobs_s) + threadIdx.x * enc_lane_stride(nb);
    const EncRun r = runs[ri];
    if (nb == 1) encode_run<1, MODE>(r, P, res + ri);
    else if (nb == 2) encode_run<2, MODE>(r, P, res + ri);
    else encode_run<4, MODE>(r, P, res + ri);
}

// raw blocks: the RAW planes of coded runs, and every plane of whole-raw
// runs (body = [1] + raw samples); one CTA per (run, plane)
__global__ void enc_raw_blocks_kernel(const EncRun* __restrict__ runs, const EncResult* __restrict__ res,
                                      const uint32_t* __restrict__ plane_prefix, int nruns, uint32_t nplanes) {
    for (uint32_t g = blockIdx.x; g < nplanes; g += gridDim.x) {
        int lo = 0, hi = nruns;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (plane_prefix[mid] <= g) lo = mid; else hi = mid;
        }
        const EncRun r = runs[lo];
        const uint32_t f = g - plane_prefix[lo];
        const uint64_t pb = (uint64_t)r.w * r.h * (r.bits / 8);
        uint8_t* dst;
        if (res[lo].whole_raw) {
            dst = r.body + 1 + f * pb;
            if (f == 0 && threadIdx.x == 0) r.body[0] = 1;
        } else {
            if (f == 0 && threadIdx.x == 0) r.body[0] = 0;
            if (r.body[1 + f] != 1) continue;
            dst = r.body + r.blk_off[f];
        }
        const uint8_t* src = r.samples + f * pb;
        for (uint64_t i = threadIdx.x; i < pb; i += blockDim.x) dst[i] = src[i];
    }
}

void launch_rc_encode(const EncRun* d_runs, const uint32_t* d_order, const int* n_per_class,
                      EncResult* d_res, const uint32_t* d_plane_prefix, int nruns, uint32_t nplanes,
                      cudaStream_t s) {
    EncClasses c;
    int nbmax = 0, off = 0, total = 0;
    for (int k = 0; k < 3; k++) total += n_per_class[k];
    // runs per warp: one while there are at most ~2 warps per SM sub-partition
    const char* ev = getenv("GSV_ENC_LANES");  // dev override
    int lanes = ev ? atoi(ev) : (total + 148 * 8 - 1) / (148 * 8);
    lanes = lanes < 1 ? 1 : (lanes > kEncRPW ? kEncRPW : lanes);
    c.lanes = lanes;
    c.blk[0] = 0;
    for (int k = 0; k < 3; k++) {
        c.n[k] = n_per_class[k];
        c.off[k] = off;
        off += c.n[k];
        c.blk[k + 1] = c.blk[k] + (c.n[k] + lanes - 1) / lanes;
        if (c.n[k] > 0) nbmax = 1 << k;
    }
    if (c.blk[3] == 0) return;
    const size_t smem = (size_t)enc_lane_stride(nbmax) * lanes;
    // renormalisation: 2 deferred (default), 1 branchy, 0 predicated (dev: GSV_ENC_MODE)
    const char* em = getenv("GSV_ENC_MODE");
    const int mode = em ? atoi(em) : 2;
#define GSV_ENC_LAUNCH(M)                                                                               \
    cudaFuncSetAttribute(rc_encode_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    rc_encode_kernel<M><<<c.blk[3], kEncRPW, smem, s>>>(d_runs, d_order, c, d_res)
    if (mode == 0) {
        GSV_ENC_LAUNCH(0);
    } else if (mode == 1) {
        GSV_ENC_LAUNCH(1);
    } else {
        GSV_ENC_LAUNCH(2);
    }
#undef GSV_ENC_LAUNCH
    if (nplanes) enc_raw_blocks_kernel<<<nplanes < 148 * 8 ? nplanes : 148 * 8, 256, 0, s>>>(
        d_runs, d_res, d_plane_prefix, nruns, nplanes);
}

}  // namespace gsv
