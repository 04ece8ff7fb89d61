// Adaptive binary range decoder for codec-1 runs (_rc.py:121-155
// decode_bittree, _rc.py:282-328 plane_from_residuals / unzigzag,
// codec.py:183-223 _decode_reference_body).
//
// A run (one (group, layer, channel) payload) is strictly sequential: its
// planes share one adaptive bit-tree model and every plane is predicted from
// the previous one.  Parallelism is therefore across runs: one lane per run,
// RPW runs of the same sample width per warp in lock-step, one warp per CTA
// so the warps spread over the SMs.  The decision chain is kept short:
//   * probabilities live in shared memory per lane as quads of nodes, and
//     the quad of the current node's grandchildren is loaded two decisions
//     before it is needed (the load latency leaves the serial chain);
//   * the coded bytes come from a big-endian 64-bit bit buffer refilled from
//     a 4-word register queue of aligned loads issued ~16 bytes ahead, and
//     the (at most two) renormalisation shifts per decision are branch-free;
//   * residual reconstruction works a 32-bit word (4/NB samples) at a time,
//     reading the previous plane and writing the output as aligned words;
//   * (variant 3, the default) a byte whose leading M decisions all take the
//     zero branch is recognised with M multiplies and one compare instead of
//     M full decisions: the high byte of 16-bit position residuals (M = 8)
//     and the top nibble of 8-bit residuals (M = 4), exact fallback otherwise.
// RAW-mode planes of these runs are first copied to 16-B aligned storage so
// that every predictor plane is aligned.
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "gsv_internal.h"

namespace gsv {

constexpr int kRPW = 32;  // runs per warp

// dev statistics: bytes redone on the careful path
__device__ unsigned long long g_rc_slow_bytes;
// dev profile (tools/rc_time.py): when set, per decoded run (run id, clock64
// cycles from the run's first plane to its last), indexed like rc_runs
__device__ unsigned long long* g_rc_prof;

__global__ void copy_planes_kernel(const CopyJob* __restrict__ jobs, int njobs) {
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const CopyJob cj = jobs[j];
        for (uint32_t i = threadIdx.x; i < cj.bytes; i += blockDim.x) cj.dst[i] = __ldg(cj.src + i);
        // the padding up to the next word: the next plane's decoder reads its
        // predictor a word at a time (the bytes past the plane are not used,
        // but they are defined -- compute-sanitizer initcheck)
        const uint32_t pad = (4u - (cj.bytes & 3u)) & 3u;
        if (threadIdx.x < pad) cj.dst[cj.bytes + threadIdx.x] = 0;
    }
}

void launch_copy_planes(const CopyJob* jobs, int njobs, cudaStream_t s) {
    if (njobs <= 0) return;
    copy_planes_kernel<<<min(njobs, 148 * 8), 256, 0, s>>>(jobs, njobs);
}

// Coded bytes as a big-endian bit buffer: the next byte sits in bits 63..56
// of `bb`, so a renormalisation by `sh` (0, 8 or 16) bits is one funnel
// shift into `code` plus a 64-bit shift of `bb`.  `bb` is refilled 32 bits
// at a time from a lane-private ring of 4 x 16 B in shared memory that
// cp.async keeps 3 chunks ahead of the read position.  (A queue of loaded
// registers was slower: the compiler's loop-carried copies read each load
// right after issuing it, so every refill waited out a global load; the
// async copies never tie a register to an in-flight load.)  Bytes past the
// block read as zero (_rc.py:129,150) and are never fetched.
constexpr uint32_t kRingBytes = 64;  // per lane

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

struct CodedStream {
    const uint8_t* gp;    // next 16-B chunk (global, aligned) to fetch
    const uint8_t* gend;  // one past the last chunk holding a byte of the block
    uint32_t ring;        // this lane's ring (shared address)
    uint32_t rpos;        // ring offset of the next word to take
    uint64_t bb;
    int32_t nbits;        // valid bits in bb
    int32_t left;         // stream bytes not yet moved into bb (<= 0: zero fill)

    // one 16-B chunk into ring slot `slot` (zero-filled past the block)
    __device__ __forceinline__ void fetch(uint32_t slot) {
        const bool in = gp < gend;
        const uint8_t* src = in ? gp : gend - 16;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n\tcp.async.commit_group;" ::"r"(ring + slot),
                     "l"(src), "r"(in ? 16 : 0)
                     : "memory");
        gp += 16;
    }
    __device__ __forceinline__ uint32_t take_word() {
        const uint32_t w = lds_u32(ring + rpos);
        rpos = (rpos + 4) & (kRingBytes - 1);
        if ((rpos & 15) == 0) {  // a chunk is used up: refetch 4 chunks ahead into its slot
            fetch((rpos - 16) & (kRingBytes - 1));
            // the chunk being entered was fetched 3 commits ago
            asm volatile("cp.async.wait_group 3;" ::: "memory");
        }
        return w;
    }
    // big-endian word with only its first m bytes kept
    __device__ __forceinline__ static uint32_t be_keep(uint32_t w_le, int32_t m) {
        const uint32_t be = __byte_perm(w_le, 0u, 0x0123);
        return m >= 4 ? be : (m > 0 ? be & ~(0xFFFFFFFFu >> (8 * m)) : 0u);
    }
    __device__ __forceinline__ void init(const uint8_t* block, uint32_t len, uint32_t ring_addr) {
        finish();  // no copy of the previous plane may still land in the ring
        const uintptr_t s = reinterpret_cast<uintptr_t>(block) + 1;  // byte 0 is always zero
        const uintptr_t e = reinterpret_cast<uintptr_t>(block) + (len ? len : 1);  // block end (exclusive)
        gp = reinterpret_cast<const uint8_t*>(s & ~uintptr_t(15));
        gend = reinterpret_cast<const uint8_t*>((e + 15) & ~uintptr_t(15));
        ring = ring_addr;
        for (uint32_t c = 0; c < 4; c++) fetch(16 * c);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        const int k = (int)(s & 15);
        rpos = (uint32_t)(k & ~3);
        left = (int32_t)len - 1;
        const int b = k & 3, nb = 4 - b;
        const uint32_t be = __byte_perm(take_word(), 0u, 0x0123) << (8 * b);  // first nb bytes on top
        const int32_t m = left < nb ? left : nb;
        const uint32_t kept = m >= 4 ? be : (m > 0 ? be & ~(0xFFFFFFFFu >> (8 * m)) : 0u);
        left -= nb;
        bb = (uint64_t)kept << 32;
        nbits = 8 * nb;
        refill();
    }
    __device__ __forceinline__ void refill() {
        if (nbits <= 32) {
            const uint32_t w = be_keep(take_word(), left);
            left -= 4;
            bb |= (uint64_t)w << (32 - nbits);
            nbits += 32;
        }
    }
    __device__ __forceinline__ uint32_t take32() {  // requires nbits >= 32
        const uint32_t v = (uint32_t)(bb >> 32);
        bb <<= 32;
        nbits -= 32;
        return v;
    }
    // drain the async copies of a finished plane (the ring is reused)
    __device__ __forceinline__ void finish() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
};

// Probabilities: lane-private, tree after tree, node n of a tree at byte
// offset 4n (so node addresses are one LEA and the quad of grandchildren
// 4c..4c+3 of node c is one aligned 128-bit load at offset 16c); lanes are
// kLaneStride apart, skewed by 16 B so that the lanes' quad loads spread over
// the banks.  At node c the quad c holds its four grandchildren: one load
// issued at decision k delivers every probability decision k+1 can need, so
// the load has two decisions to land and never sits on the bit-serial chain.
// Shared accesses are volatile PTX so the compiler neither converts the
// speculative loads into bit-dependent ones nor reorders them around the
// probability stores.
constexpr uint32_t kTreeBytes = 256u * 4u;
__host__ __device__ constexpr uint32_t lane_stride(int nb) { return (uint32_t)nb * kTreeBytes + 16u; }

__device__ __forceinline__ uint4 lds_quad(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint32_t node_addr(uint32_t tree, uint32_t node) { return tree + node * 4u; }

// Adaptive update of one node (_rc.py:140-146): bit 0: p += (4096 - p) >> 4,
// bit 1: p -= p >> 4.  Both are p + ((K - p) >> 4) with an arithmetic shift,
// K = 4096 or 15 (floor((15 - p) / 16) == -floor(p / 16) for integer p).
__device__ __forceinline__ uint32_t adapt(uint32_t p, bool bit) {
    return p + (uint32_t)(((int32_t)(bit ? 15u : 4096u) - (int32_t)p) >> 4);
}

// 8 decisions of one byte on tree T, careful path: every decision stores its
// node and keeps >= 32 buffered bits (at most 32 are consumed per two
// decisions).  q0 holds quad 0 of T on entry (node 1 and its children) and
// quad 0 of tree Tn on exit.
__device__ __forceinline__ uint32_t decode_byte_slow(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                     uint32_t& code, CodedStream& cs) {
    atomicAdd(&g_rc_slow_bytes, 1ull);
    uint32_t ctx = 1;
    uint32_t p = q0.y;  // node 1
    uint4 cq = q0;      // quad holding the children of ctx
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint4 nq = make_uint4(0u, 0u, 0u, 0u);
        if (k < 6) nq = lds_quad(T + ctx * 16u);  // grandchildren of ctx
        const uint32_t c0 = (ctx & 1) ? cq.z : cq.x;
        const uint32_t c1 = (ctx & 1) ? cq.w : cq.y;
        const uint32_t bound = (rng >> 12) * p;
        const bool bit = code >= bound;
        code = bit ? code - bound : code;
        rng = bit ? rng - bound : bound;
        sts_u32(node_addr(T, ctx), adapt(p, bit));
        ctx = 2 * ctx + (bit ? 1u : 0u);
        p = bit ? c1 : c0;
        cq = nq;
        // renormalise: rng >= 2^15 after any decision, so shift by 0, 8 or 16
        const uint32_t sh = rng < (1u << 24) ? (rng < (1u << 16) ? 16u : 8u) : 0u;
        code = __funnelshift_l((uint32_t)(cs.bb >> 32), code, sh);
        rng <<= sh;
        cs.bb <<= sh;
        cs.nbits -= (int32_t)sh;
        if (k & 1) cs.refill();
    }
    q0 = lds_quad(Tn);  // after this byte's stores (Tn may be T)
    return ctx & 0xFFu;
}

// Fast path.  Within one byte the decisions only ever shift whole bytes in
// (renormalisation by 8; a shift by 16 needs rng < 2^16 and is left to the
// careful path), and the next four stream bytes sit in `bhi`, so the
// renormalisation is a predicated byte permute of `code` with the next byte
// and a predicated shift of `rng`; the next (rng >> 12) is selected from two
// shifts computed beside the compare.  The bit-serial chain per decision is
// then multiply -> compare -> select rng -> compare 2^24 -> select (rng >> 12).
// The 8 probability stores are deferred to the end of the byte (so the
// careful path can redo the byte from untouched state when it consumed more
// than 4 bytes or needed a 16-bit shift: both are rare).  Multi-byte samples
// alternate trees, so q0 of the next tree is loaded during this byte; for
// one-byte samples the next root quad is this tree's, patched in registers.
// a shift the compiler cannot fold into a select of shift amounts (which
// would put the select before the shift on the serial chain)
template <int S>
__device__ __forceinline__ uint32_t shr_opaque(uint32_t x) {
    uint32_t y;
    asm("shr.b32 %0, %1, %2;" : "=r"(y) : "r"(x), "n"(S));
    return y;
}

template <bool SAME_TREE>
__device__ __forceinline__ uint32_t decode_byte(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                uint32_t& code, CodedStream& cs) {
    const uint32_t rng0 = rng, code0 = code;
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);  // next 4 stream bytes, first in bits 31..24
    uint32_t ctx = 1, sel = 0x2107u;               // byte_perm: (code << 8) | next stream byte
    uint32_t p = q0.y;
    uint4 cq = q0;
    uint4 qn = q0;
    uint32_t pn[8], na[8];
    uint32_t a = rng >> 12;
    bool wide = false;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint4 nq = make_uint4(0u, 0u, 0u, 0u);
        if (k < 6) nq = lds_quad(T + ctx * 16u);
        if (!SAME_TREE && k == 6) qn = lds_quad(Tn);
        na[k] = node_addr(T, ctx);
        const uint32_t c0 = (ctx & 1) ? cq.z : cq.x;
        const uint32_t c1 = (ctx & 1) ? cq.w : cq.y;
        const uint32_t bound = a * p;
        const bool bit = code >= bound;
        const uint32_t r = bit ? rng - bound : bound;
        code = bit ? code - bound : code;
        pn[k] = adapt(p, bit);
        ctx = 2 * ctx + (bit ? 1u : 0u);
        p = bit ? c1 : c0;
        cq = nq;
        const bool lt24 = r < (1u << 24);
        wide |= r < (1u << 16);
        a = lt24 ? shr_opaque<4>(r) : shr_opaque<12>(r);  // both shifts beside the compare
        rng = lt24 ? (r << 8) : r;
        code = lt24 ? __byte_perm(code, bhi, sel) : code;
        sel -= lt24 ? 1u : 0u;
    }
    const uint32_t used = 0x2107u - sel;  // stream bytes shifted in
    if (wide || used > 4u) {             // rare: redo carefully (nothing was stored)
        rng = rng0;
        code = code0;
        return decode_byte_slow(T, Tn, q0, rng, code, cs);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) sts_u32(na[k], pn[k]);
    if (SAME_TREE) {
        const bool b0 = (ctx >> 7) & 1u;  // first decision: node 2 or 3 was updated second
        qn.y = pn[0];
        qn.z = b0 ? q0.z : pn[1];
        qn.w = b0 ? pn[1] : q0.w;
    }
    q0 = qn;
    cs.bb <<= 8 * used;
    cs.nbits -= (int32_t)(8 * used);
    cs.refill();
    return ctx & 0xFFu;
}

// Variant 2: the same fast path with the decision step written in PTX so
// that the renormalisation, the code update and the node-address walk stay
// predicated single instructions (the compiler otherwise expands selects into
// two instructions).  Node addresses are walked directly: child = 2 * node -
// T + 4 * bit (byte offsets, node n at T + 4n), grandchild quad at 4 * node -
// 3T.
template <bool SAME_TREE>
__device__ __forceinline__ uint32_t decode_byte_v2(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                   uint32_t& code, CodedStream& cs) {
    const uint32_t rng0 = rng, code0 = code;
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);
    uint32_t sel = 0x2107u, rmin = 0xFFFFFFFFu;
    uint32_t p = q0.y;
    uint4 cq = q0;
    uint4 qn = q0;
    uint32_t pn[8], na[8];
    uint32_t a = rng >> 12;
    uint32_t node = T + 4u;                // node 1
    const uint32_t m3T = 0u - 3u * T, c0T = 0u - T, c1T = 4u - T;
    uint32_t pbit = 1u;                    // ctx & 1 of the current node (node 1: odd)
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint4 nq = make_uint4(0u, 0u, 0u, 0u);
        if (k < 6) nq = lds_quad(4u * node + m3T);
        if (!SAME_TREE && k == 6) qn = lds_quad(Tn);
        na[k] = node;
        const uint32_t c0 = pbit ? cq.z : cq.x;
        const uint32_t c1 = pbit ? cq.w : cq.y;
        uint32_t bitv, nnode;
        asm("{\n\t"
            ".reg .pred pb, pl;\n\t"
            ".reg .u32 bnd, r1, r, t4, t12, K, d, off;\n\t"
            "mul.lo.u32 bnd, %0, %9;\n\t"
            "setp.ge.u32 pb, %2, bnd;\n\t"
            "sub.u32 r1, %1, bnd;\n\t"
            "selp.u32 r, r1, bnd, pb;\n\t"
            "@pb sub.u32 %2, %2, bnd;\n\t"
            "setp.lt.u32 pl, r, 16777216;\n\t"
            "min.u32 %4, %4, r;\n\t"
            "shr.u32 t4, r, 4;\n\t"
            "shr.u32 t12, r, 12;\n\t"
            "selp.u32 %0, t4, t12, pl;\n\t"
            "@pl shl.b32 r, r, 8;\n\t"
            "@pl prmt.b32 %2, %2, %10, %3;\n\t"
            "@pl sub.u32 %3, %3, 1;\n\t"
            "mov.u32 %1, r;\n\t"
            "selp.u32 K, 15, 4096, pb;\n\t"
            "sub.s32 d, K, %9;\n\t"
            "shr.s32 d, d, 4;\n\t"
            "add.u32 %5, %9, d;\n\t"
            "selp.u32 %6, %12, %11, pb;\n\t"
            "selp.u32 off, %14, %13, pb;\n\t"
            "mad.lo.u32 %7, %15, 2, off;\n\t"
            "selp.u32 %8, 1, 0, pb;\n\t"
            "}"
            : "+r"(a), "+r"(rng), "+r"(code), "+r"(sel), "+r"(rmin), "=r"(pn[k]), "=r"(p), "=r"(nnode),
              "=r"(bitv)
            : "r"(p), "r"(bhi), "r"(c0), "r"(c1), "r"(c0T), "r"(c1T), "r"(node));
        node = nnode;
        pbit = bitv;
        cq = nq;
    }
    const uint32_t used = 0x2107u - sel;
    if (rmin < (1u << 16) || used > 4u) {
        rng = rng0;
        code = code0;
        return decode_byte_slow(T, Tn, q0, rng, code, cs);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) sts_u32(na[k], pn[k]);
    const uint32_t ctx = (node - T) >> 2;  // 256 + byte value
    if (SAME_TREE) {
        const bool b0 = (ctx >> 7) & 1u;
        qn.y = pn[0];
        qn.z = b0 ? q0.z : pn[1];
        qn.w = b0 ? pn[1] : q0.w;
    }
    q0 = qn;
    cs.bb <<= 8 * used;
    cs.nbits -= (int32_t)(8 * used);
    cs.refill();
    return ctx & 0xFFu;
}

// fixed point of the zero-branch adaptation p += (4096 - p) >> 4
constexpr uint32_t kZeroSat = 4081u;

// Variant 3: zero-prefix test.  Along the all-zero path of a bit tree
// (nodes 1, 2, 4, ..., 2^(M-1)) a 0 decision leaves `code` alone and sets
// rng = bound, so the nested intervals [0, bound_k) shrink and the first M
// decisions are all 0 iff the code (shifted by the renormalisation bytes
// taken before decision M-1, which preserves the order of code and bound)
// lies below the last bound.  That bound chain needs only rng and the M
// zero-path probabilities, not the bits, so M decisions cost M multiplies
// and one compare.  Position residuals (2-byte samples) have a zero high
// byte (M = 8: the whole byte) and 1-byte residuals are small (M = 4); when
// the test fails the byte is decoded by variant 2 from the untouched state.
template <int M, bool SAME_TREE>
__device__ __forceinline__ uint32_t decode_byte_v3(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                   uint32_t& code, CodedStream& cs, bool* sat = nullptr) {
    static_assert(M >= 2 && M <= 8, "zero prefix length");
    if (sat) *sat = false;  // set again below when the zero path ends saturated
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);
    uint32_t z[M + 1];  // zero-path probabilities (z[M]: the node decision M starts at)
    z[0] = q0.y;
    z[1] = q0.z;
#pragma unroll
    for (int k = 2; k <= M && k < 8; k++) z[k] = lds_u32(T + 4u * (1u << k));
    uint4 qn = q0, cq = make_uint4(0u, 0u, 0u, 0u), nq0 = cq;
    if (!SAME_TREE) qn = lds_quad(Tn);
    if (M < 8) cq = lds_quad(T + 16u * (1u << (M - 1)));  // children of node 2^M
    if (M < 6) nq0 = lds_quad(T + 16u * (1u << M));       // its grandchildren
    uint32_t a = rng >> 12, rmin = 0xFFFFFFFFu, S = 0, bound = 0;
#pragma unroll
    for (int k = 0; k < M; k++) {
        bound = a * z[k];
        rmin = min(rmin, bound);
        const bool lt24 = bound < (1u << 24);
        a = lt24 ? shr_opaque<4>(bound) : shr_opaque<12>(bound);
        if (k < M - 1) S += lt24 ? 1u : 0u;
    }
    // (code:bhi) << 8S must stay below bound as a 64-bit value: no code
    // bits may be shifted out (the zero path would have failed earlier)
    if (__funnelshift_lc(code, 0u, 8u * S) != 0u || !(__funnelshift_lc(bhi, code, 8u * S) < bound) ||
        rmin < (1u << 16) || S > 3u)
        return decode_byte_v2<SAME_TREE>(T, Tn, q0, rng, code, cs);
    const uint32_t rng0 = rng, code0 = code;
    const bool lt24 = bound < (1u << 24);
    S += lt24 ? 1u : 0u;
    rng = lt24 ? bound << 8 : bound;
    code = __funnelshift_lc(bhi, code, 8u * S);
    uint32_t pn[8], na[8];
#pragma unroll
    for (int k = 0; k < M; k++) {
        pn[k] = z[k] + ((4096u - z[k]) >> 4);
        na[k] = T + 4u * (1u << k);
    }
    uint32_t sel = 0x2107u - S;
    uint32_t node = T + 4u * (1u << (M < 8 ? M : 0));
    if (M < 8) {
        uint32_t p = z[M < 8 ? M : 0];
        const uint32_t m3T = 0u - 3u * T, c0T = 0u - T, c1T = 4u - T;
        uint32_t pbit = 0u;
#pragma unroll
        for (int k = M; k < 8; k++) {
            uint4 nq = make_uint4(0u, 0u, 0u, 0u);
            if (k == M) nq = nq0;
            else if (k < 6) nq = lds_quad(4u * node + m3T);
            na[k] = node;
            const uint32_t c0 = pbit ? cq.z : cq.x;
            const uint32_t c1 = pbit ? cq.w : cq.y;
            uint32_t bitv, nnode;
            asm("{\n\t"
                ".reg .pred pb, pl;\n\t"
                ".reg .u32 bnd, r1, r, t4, t12, K, d, off;\n\t"
                "mul.lo.u32 bnd, %0, %9;\n\t"
                "setp.ge.u32 pb, %2, bnd;\n\t"
                "sub.u32 r1, %1, bnd;\n\t"
                "selp.u32 r, r1, bnd, pb;\n\t"
                "@pb sub.u32 %2, %2, bnd;\n\t"
                "setp.lt.u32 pl, r, 16777216;\n\t"
                "min.u32 %4, %4, r;\n\t"
                "shr.u32 t4, r, 4;\n\t"
                "shr.u32 t12, r, 12;\n\t"
                "selp.u32 %0, t4, t12, pl;\n\t"
                "@pl shl.b32 r, r, 8;\n\t"
                "@pl prmt.b32 %2, %2, %10, %3;\n\t"
                "@pl sub.u32 %3, %3, 1;\n\t"
                "mov.u32 %1, r;\n\t"
                "selp.u32 K, 15, 4096, pb;\n\t"
                "sub.s32 d, K, %9;\n\t"
                "shr.s32 d, d, 4;\n\t"
                "add.u32 %5, %9, d;\n\t"
                "selp.u32 %6, %12, %11, pb;\n\t"
                "selp.u32 off, %14, %13, pb;\n\t"
                "mad.lo.u32 %7, %15, 2, off;\n\t"
                "selp.u32 %8, 1, 0, pb;\n\t"
                "}"
                : "+r"(a), "+r"(rng), "+r"(code), "+r"(sel), "+r"(rmin), "=r"(pn[k]), "=r"(p), "=r"(nnode),
                  "=r"(bitv)
                : "r"(p), "r"(bhi), "r"(c0), "r"(c1), "r"(c0T), "r"(c1T), "r"(node));
            node = nnode;
            pbit = bitv;
            cq = nq;
        }
        if (rmin < (1u << 16) || 0x2107u - sel > 4u) {
            rng = rng0;
            code = code0;
            return decode_byte_slow(T, Tn, q0, rng, code, cs);
        }
    }
    const uint32_t used = 0x2107u - sel;
#pragma unroll
    for (int k = 0; k < 8; k++) sts_u32(na[k], pn[k]);
    if (sat) {
        bool all = true;
#pragma unroll
        for (int k = 0; k < M; k++) all = all && pn[k] == kZeroSat;
        *sat = all;
    }
    const uint32_t ctx = M < 8 ? (node - T) >> 2 : 256u;
    if (SAME_TREE) {  // first decision was 0: nodes 1 and 2 were updated
        qn.y = pn[0];
        qn.z = pn[1];
    }
    q0 = qn;
    cs.bb <<= 8 * used;
    cs.nbits -= (int32_t)(8 * used);
    cs.refill();
    return ctx & 0xFFu;
}

// Whole-byte zero test (M = 8, next tree Tn != T): true and the state
// advanced past a zero byte, or false and nothing touched (the caller then
// decodes the byte with its single variant-2 instance).
__device__ __forceinline__ bool zero_byte(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng, uint32_t& code,
                                          CodedStream& cs, bool* sat = nullptr) {
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);
    uint32_t z[8];
    z[0] = q0.y;
    z[1] = q0.z;
#pragma unroll
    for (int k = 2; k < 8; k++) z[k] = lds_u32(T + 4u * (1u << k));
    uint32_t a = rng >> 12, rmin = 0xFFFFFFFFu, S = 0, bound = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        bound = a * z[k];
        rmin = min(rmin, bound);
        const bool lt24 = bound < (1u << 24);
        a = lt24 ? shr_opaque<4>(bound) : shr_opaque<12>(bound);
        if (k < 7) S += lt24 ? 1u : 0u;
    }
    if (__funnelshift_lc(code, 0u, 8u * S) != 0u || !(__funnelshift_lc(bhi, code, 8u * S) < bound) ||
        rmin < (1u << 16) || S > 3u)
        return false;
    const uint4 qn = lds_quad(Tn);
    const bool lt24 = bound < (1u << 24);
    S += lt24 ? 1u : 0u;
    rng = lt24 ? bound << 8 : bound;
    code = __funnelshift_lc(bhi, code, 8u * S);
    bool all = true;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const uint32_t pk = z[k] + ((4096u - z[k]) >> 4);
        all = all && pk == kZeroSat;
        sts_u32(T + 4u * (1u << k), pk);
    }
    if (sat) *sat = all;
    q0 = qn;
    cs.bb <<= 8 * S;
    cs.nbits -= (int32_t)(8 * S);
    cs.refill();
    return true;
}

// One full binary decision (the variant-2 step) as a function: bound,
// compare, interval update, renormalisation by a predicated byte permute,
// adapted probability, the child's probability and node address.
__device__ __forceinline__ void rc_step(uint32_t& a, uint32_t& rng, uint32_t& code, uint32_t& sel, uint32_t& rmin,
                                        uint32_t& pn, uint32_t& p, uint32_t& node, uint32_t& pbit, uint32_t bhi,
                                        uint32_t c0, uint32_t c1, uint32_t c0T, uint32_t c1T) {
    uint32_t bitv, nnode;
    asm("{\n\t"
        ".reg .pred pb, pl;\n\t"
        ".reg .u32 bnd, r1, r, t4, t12, K, d, off;\n\t"
        "mul.lo.u32 bnd, %0, %9;\n\t"
        "setp.ge.u32 pb, %2, bnd;\n\t"
        "sub.u32 r1, %1, bnd;\n\t"
        "selp.u32 r, r1, bnd, pb;\n\t"
        "@pb sub.u32 %2, %2, bnd;\n\t"
        "setp.lt.u32 pl, r, 16777216;\n\t"
        "min.u32 %4, %4, r;\n\t"
        "shr.u32 t4, r, 4;\n\t"
        "shr.u32 t12, r, 12;\n\t"
        "selp.u32 %0, t4, t12, pl;\n\t"
        "@pl shl.b32 r, r, 8;\n\t"
        "@pl prmt.b32 %2, %2, %10, %3;\n\t"
        "@pl sub.u32 %3, %3, 1;\n\t"
        "mov.u32 %1, r;\n\t"
        "selp.u32 K, 15, 4096, pb;\n\t"
        "sub.s32 d, K, %9;\n\t"
        "shr.s32 d, d, 4;\n\t"
        "add.u32 %5, %9, d;\n\t"
        "selp.u32 %6, %12, %11, pb;\n\t"
        "selp.u32 off, %14, %13, pb;\n\t"
        "mad.lo.u32 %7, %15, 2, off;\n\t"
        "selp.u32 %8, 1, 0, pb;\n\t"
        "}"
        : "+r"(a), "+r"(rng), "+r"(code), "+r"(sel), "+r"(rmin), "=r"(pn), "=r"(p), "=r"(nnode), "=r"(bitv)
        : "r"(p), "r"(bhi), "r"(c0), "r"(c1), "r"(c0T), "r"(c1T), "r"(node));
    node = nnode;
    pbit = bitv;
}

// Variant 4: the zero-prefix tests of variant 3 once their path is
// SATURATED.  A zero decision moves p to p + ((4096 - p) >> 4), whose fixed
// point is 4081; after ~50 zero prefixes in a row (position high bytes are
// always zero, 8-bit residuals always have a zero top nibble) every node on
// the zero path holds 4081 and stays there.  A lane-private flag records
// that state, and then M zero decisions are exactly: bounds b_k = (b_{k-1} >>
// 12) * 4081 while no renormalisation intervenes (b_{M-2} >= 2^24: bounds
// decrease), and the path is taken iff code < b_{M-1}.  That is M
// multiply-shift pairs and two compares -- no probability loads, no
// adaptation, no stores.  Anything else (not saturated, a bound below 2^24
// before the last decision, the code above the bound) goes to the exact
// variant-3 path, which also re-derives the flag.
__device__ __forceinline__ bool zero_byte_sat(uint32_t Tn, uint4& q0, uint32_t& rng, uint32_t& code,
                                              CodedStream& cs) {
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);
    uint32_t b = shr_opaque<12>(rng) * kZeroSat, bp = b;
#pragma unroll
    for (int k = 1; k < 8; k++) {
        bp = b;
        b = shr_opaque<12>(b) * kZeroSat;
    }
    if (!(bp >= (1u << 24) && code < b)) return false;
    q0 = lds_quad(Tn);
    const uint32_t S = b < (1u << 24) ? 1u : 0u;  // b > 2^16: one renormalisation at most
    rng = S ? b << 8 : b;
    code = S ? __byte_perm(code, bhi, 0x2107u) : code;  // (code << 8) | next stream byte
    cs.bb <<= 8 * S;
    cs.nbits -= (int32_t)(8 * S);
    cs.refill();
    return true;
}

// 1-byte samples: a saturated 4-decision zero prefix (top nibble), then the
// 4 low decisions as variant 2 does them; otherwise variant 3.
__device__ __forceinline__ uint32_t decode_byte_v4(uint32_t T, uint4& q0, uint32_t& rng, uint32_t& code,
                                                   CodedStream& cs, bool& sat) {
    constexpr int M = 4;
    if (sat) {
        const uint32_t bhi = (uint32_t)(cs.bb >> 32);
        uint32_t p = lds_u32(T + 4u * (1u << M));           // node 16
        uint4 cq = lds_quad(T + 16u * (1u << (M - 1)));     // its children 32, 33
        uint4 nq = lds_quad(T + 16u * (1u << M));           // its grandchildren 64..67
        uint32_t b = shr_opaque<12>(rng) * kZeroSat, bp = b;
#pragma unroll
        for (int k = 1; k < M; k++) {
            bp = b;
            b = shr_opaque<12>(b) * kZeroSat;
        }
        if (bp >= (1u << 24) && code < b) {
            const uint32_t rng0 = rng, code0 = code;
            const uint32_t S = b < (1u << 24) ? 1u : 0u;
            rng = S ? b << 8 : b;
            code = S ? __byte_perm(code, bhi, 0x2107u) : code;
            uint32_t a = rng >> 12, sel = 0x2107u - S, rmin = 0xFFFFFFFFu;
            uint32_t node = T + 4u * (1u << M), pbit = 0u, pn[8 - M], na[8 - M];
            const uint32_t m3T = 0u - 3u * T, c0T = 0u - T, c1T = 4u - T;
#pragma unroll
            for (int k = M; k < 8; k++) {
                uint4 nn = make_uint4(0u, 0u, 0u, 0u);
                if (k == M) nn = nq;
                else if (k < 6) nn = lds_quad(4u * node + m3T);
                na[k - M] = node;
                const uint32_t c0 = pbit ? cq.z : cq.x, c1 = pbit ? cq.w : cq.y;
                rc_step(a, rng, code, sel, rmin, pn[k - M], p, node, pbit, bhi, c0, c1, c0T, c1T);
                cq = nn;
            }
            const uint32_t used = 0x2107u - sel;
            if (rmin < (1u << 16) || used > 4u) {  // rare: the careful path redoes the byte
                rng = rng0;
                code = code0;
                sat = false;
                return decode_byte_slow(T, T, q0, rng, code, cs);
            }
#pragma unroll
            for (int k = 0; k < 8 - M; k++) sts_u32(na[k], pn[k]);
            cs.bb <<= 8 * used;
            cs.nbits -= (int32_t)(8 * used);
            cs.refill();
            return ((node - T) >> 2) & 0xFFu;  // q0 unchanged: nodes 1 and 2 still hold 4081
        }
    }
    return decode_byte_v3<M, true>(T, T, q0, rng, code, cs, &sat);
}

template <int V, bool SAME_TREE>
__device__ __forceinline__ uint32_t decode_byte_v(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                  uint32_t& code, CodedStream& cs) {
    if constexpr (V >= 2) return decode_byte_v2<SAME_TREE>(T, Tn, q0, rng, code, cs);
    else return decode_byte<SAME_TREE>(T, Tn, q0, rng, code, cs);
}

template <int V, int NB, bool PREV>
__device__ __forceinline__ void decode_plane(uint32_t P, uint32_t R, const PlaneRef& pr,
                                             const uint32_t* __restrict__ prev,
                                             uint32_t* __restrict__ out, uint32_t hw, uint32_t w, bool& sat) {
    constexpr int SPW = 4 / NB;  // samples per 32-bit word
    constexpr uint32_t mask = NB == 4 ? 0xFFFFFFFFu : ((1u << (8 * NB)) - 1u);
    constexpr uint32_t def = 128u << (8 * NB - 8);
    CodedStream cs;
    cs.init(pr.coded, pr.coded_len, R);
    uint32_t code = cs.take32();
    cs.refill();
    uint32_t rng = 0xFFFFFFFFu;
    uint4 q0 = lds_quad(P);                  // root quad of tree 0
    // previous plane, 4 words at a time, one group ahead (planes are 16-B
    // aligned with slack after them, so the read-ahead stays in bounds)
    const uint4* pp = reinterpret_cast<const uint4*>(prev);
    uint4 cur = make_uint4(0u, 0u, 0u, 0u), nxt = cur;
    if (PREV) cur = __ldg(pp);
    uint32_t left = 0, above = 0, x = 0;
    const uint32_t nwords = (hw * NB + 3) / 4;
    uint32_t idx = 0;
    for (uint32_t g = 0; g < nwords; g += 4) {
        if (PREV) nxt = __ldg(pp + g / 4 + 1);
#pragma unroll 1
        for (int q = 0; q < 4; q++) {  // not unrolled: the loop body must stay small in the i-cache
            const uint32_t wi = g + q;
            if (wi >= nwords) break;
            const uint32_t pw = q == 0 ? cur.x : (q == 1 ? cur.y : (q == 2 ? cur.z : cur.w));
            uint32_t ow = 0, z = 0;
            // one byte per iteration and a single inlined decoder instance,
            // so the loop body stays small in the instruction cache
            // (variant 3, 2-byte samples: one sample per iteration, the high
            // byte by the zero test with a cold variant-2 fallback)
            constexpr int BPI = (V >= 3 && NB == 2) ? 2 : 1;
#pragma unroll 1
            for (int e = 0; e < SPW * NB; e += BPI) {
                const int j = e / NB, b = e % NB;
                if (SPW > 1 && idx >= hw) break;
                const uint32_t T = P + (uint32_t)b * kTreeBytes;
                const uint32_t Tn = NB == 1 ? T : P + (uint32_t)((b + 1) % NB) * kTreeBytes;
                if (V == 4 && NB == 2) {
                    const uint32_t T1 = P + kTreeBytes;
                    z = decode_byte_v2<false>(P, T1, q0, rng, code, cs);
                    if (!(sat && zero_byte_sat(P, q0, rng, code, cs)) && !zero_byte(T1, P, q0, rng, code, cs, &sat)) {
                        z |= decode_byte_v2<false>(T1, P, q0, rng, code, cs) << 8;
                        sat = false;
                    }
                } else if (V == 4 && NB == 1) {
                    z = decode_byte_v4(T, q0, rng, code, cs, sat);
                } else if (V == 3 && NB == 2) {
                    const uint32_t T1 = P + kTreeBytes;
                    z = decode_byte_v2<false>(P, T1, q0, rng, code, cs);
                    if (!zero_byte(T1, P, q0, rng, code, cs)) z |= decode_byte_v2<false>(T1, P, q0, rng, code, cs) << 8;
                } else if (V == 3 && NB == 1) {
                    z = decode_byte_v3<4, true>(T, Tn, q0, rng, code, cs);
                } else {
                    z |= decode_byte_v<V, NB == 1>(T, Tn, q0, rng, code, cs) << (8 * b);
                }
                if (b + BPI - 1 == NB - 1) {
                    uint32_t pred;
                    if (PREV) {
                        pred = (pw >> (8 * NB * j)) & mask;
                    } else {
                        pred = x > 0 ? left : (idx > 0 ? above : def);
                    }
                    const uint32_t v = (pred + ((z >> 1) ^ (0u - (z & 1u)))) & mask;  // unzigzag
                    if (!PREV) {
                        if (x == 0) above = v;
                        left = v;
                        if (++x == w) x = 0;
                    }
                    ow |= v << (8 * NB * j);
                    idx++;
                    z = 0;
                }
            }
            out[wi] = ow;
        }
        cur = nxt;
    }
}

// ===========================================================================
// Variant 5: warp-cooperative speculative decoding.
//
// The serial chain of one run is what bounds codec 1 (a run's decisions
// depend on each other; runs are the only independent units), and a lane
// that walks the tree alone spends ~25 instructions per decision on one
// sub-partition.  Here the LANES of a warp share ONE run and decode a byte by
// speculation over its leading decisions: lane i assumes the byte starts
// with the bits of i and evaluates those decisions along its own path --
// bound, interval update, renormalisation; the bit is known, so the compare
// is only a check off the chain -- and the one lane whose assumed bits are
// the decisions the reference makes (at its first wrong bit a lane's state is
// still the true state, so its check fails there) holds the true state.  A
// ballot finds it and a shuffle hands its state to every lane.  The bit tree
// lives in REGISTERS distributed over the lanes: a lane keeps the nodes of
// its assumed path (shared nodes replicated in every lane whose path crosses
// them) and, below it, its own subtree; after each byte every lane adapts the
// copies it holds of the winner's path, so no probability goes through
// shared memory on the chain.  The tree is only written to shared memory when
// a byte needs the careful path (a 16-bit renormalisation or more than four
// stream bytes in one byte: the byte is redone there by the scalar decoder).
//   * 16-bit runs (position residuals: the longest chains): one run per warp,
//     low byte = 5 assumed bits (32 lanes) + 3 decisions each lane takes in
//     its own subtree; high byte (always zero here) by the saturated zero test
//     of variant 4, else the same speculation on its tree.
//   * 8-bit runs (residuals below 16): two runs per warp, 16 lanes each: the
//     saturated zero nibble (p = 4081 on nodes 1, 2, 4, 8) followed by 4
//     assumed bits of the low nibble; any other byte (nibble not zero, zero
//     path not saturated) takes the careful path.
// Same arithmetic, same stream bytes, same adaptation as _rc.py:121-155.

// p + ((K - p) >> 4) for a bit known as a u32 0/1 (see adapt())
__device__ __forceinline__ uint32_t adapt_u(uint32_t p, uint32_t bit) {
    return p + (uint32_t)(((int32_t)(bit ? 15u : 4096u) - (int32_t)p) >> 4);
}

// Known-bit decision: km = 0xFFFFFFFF when the assumed bit is 1, else 0;
// pk = km ? -p : p and rm = r & km (so rr = a * pk + rm is bit ? r - b : b in
// one multiply-add).  Produces rm for the next step (mask kmn) beside a.
__device__ __forceinline__ void kstep(uint32_t& a, uint32_t& rm, uint32_t& c, uint32_t& sel, uint32_t& rmin,
                                      uint32_t& bad, uint32_t& rr, uint32_t p, uint32_t pk, uint32_t km,
                                      uint32_t kmn, uint32_t bhi) {
    asm("{\n\t"
        ".reg .pred pl, pk1;\n\t"
        ".reg .u32 b, t, t4, t12, t8, m0, m1;\n\t"
        "mul.lo.u32 b, %0, %8;\n\t"
        "mad.lo.u32 %6, %0, %9, %1;\n\t"
        "set.ge.u32.u32 t, %2, b;\n\t"
        "xor.b32 t, t, %10;\n\t"
        "or.b32 %5, %5, t;\n\t"
        "setp.ne.u32 pk1, %10, 0;\n\t"
        "@pk1 sub.u32 %2, %2, b;\n\t"
        "min.u32 %4, %4, %6;\n\t"
        "setp.lt.u32 pl, %6, 16777216;\n\t"
        "shr.u32 t4, %6, 4;\n\t"
        "shr.u32 t12, %6, 12;\n\t"
        "selp.u32 %0, t4, t12, pl;\n\t"
        "shl.b32 t8, %6, 8;\n\t"
        "and.b32 m1, t8, %11;\n\t"
        "and.b32 m0, %6, %11;\n\t"
        "selp.u32 %1, m1, m0, pl;\n\t"
        "@pl mov.u32 %6, t8;\n\t"
        "@pl prmt.b32 %2, %2, %7, %3;\n\t"
        "@pl sub.u32 %3, %3, 1;\n\t"
        "}"
        : "+r"(a), "+r"(rm), "+r"(c), "+r"(sel), "+r"(rmin), "+r"(bad), "=r"(rr)
        : "r"(bhi), "r"(p), "r"(pk), "r"(km), "r"(kmn));
}

// Full decision (the bit is decided here): as rc_step, without the node walk.
__device__ __forceinline__ uint32_t fstep(uint32_t& a, uint32_t& r, uint32_t& c, uint32_t& sel, uint32_t& rmin,
                                          uint32_t& pn, uint32_t p, uint32_t bhi) {
    uint32_t bitv;
    asm("{\n\t"
        ".reg .pred pb, pl;\n\t"
        ".reg .u32 b, r1, rr, t4, t12, K, d;\n\t"
        "mul.lo.u32 b, %0, %7;\n\t"
        "setp.ge.u32 pb, %2, b;\n\t"
        "sub.u32 r1, %1, b;\n\t"
        "selp.u32 rr, r1, b, pb;\n\t"
        "@pb sub.u32 %2, %2, b;\n\t"
        "min.u32 %4, %4, rr;\n\t"
        "setp.lt.u32 pl, rr, 16777216;\n\t"
        "shr.u32 t4, rr, 4;\n\t"
        "shr.u32 t12, rr, 12;\n\t"
        "selp.u32 %0, t4, t12, pl;\n\t"
        "@pl shl.b32 rr, rr, 8;\n\t"
        "mov.u32 %1, rr;\n\t"
        "@pl prmt.b32 %2, %2, %8, %3;\n\t"
        "@pl sub.u32 %3, %3, 1;\n\t"
        "selp.u32 K, 15, 4096, pb;\n\t"
        "sub.s32 d, K, %7;\n\t"
        "shr.s32 d, d, 4;\n\t"
        "add.u32 %5, %7, d;\n\t"
        "selp.u32 %6, 1, 0, pb;\n\t"
        "}"
        : "+r"(a), "+r"(r), "+r"(c), "+r"(sel), "+r"(rmin), "=r"(pn), "=r"(bitv)
        : "r"(p), "r"(bhi));
    return bitv;
}

// Zero decision at the saturated probability 4081 (kstep with bit 0, p fixed).
__device__ __forceinline__ void zstep(uint32_t& a, uint32_t& r, uint32_t& c, uint32_t& sel, uint32_t& rmin,
                                      uint32_t& bad, uint32_t bhi) {
    asm("{\n\t"
        ".reg .pred pl;\n\t"
        ".reg .u32 b, t, t4, t12;\n\t"
        "mul.lo.u32 b, %0, 4081;\n\t"
        "set.ge.u32.u32 t, %2, b;\n\t"
        "or.b32 %5, %5, t;\n\t"
        "min.u32 %4, %4, b;\n\t"
        "setp.lt.u32 pl, b, 16777216;\n\t"
        "shr.u32 t4, b, 4;\n\t"
        "shr.u32 t12, b, 12;\n\t"
        "selp.u32 %0, t4, t12, pl;\n\t"
        "@pl shl.b32 b, b, 8;\n\t"
        "mov.u32 %1, b;\n\t"
        "@pl prmt.b32 %2, %2, %6, %3;\n\t"
        "@pl sub.u32 %3, %3, 1;\n\t"
        "}"
        : "+r"(a), "+r"(r), "+r"(c), "+r"(sel), "+r"(rmin), "+r"(bad)
        : "r"(bhi));
}

// One bit tree over 32 lanes: p[d] = node (1 << d) | (lane >> (5 - d)) (the
// lane's 5-bit path), s[0] = node 32 + lane, s[1 + b] = node 64 + 2 lane + b,
// s[3 + q] = node 128 + 4 lane + q (the lane's subtree).
struct Tree32 {
    uint32_t p[5], s[7];
};

__device__ __forceinline__ void tree32_load(Tree32& t, uint32_t T, uint32_t lane) {
#pragma unroll
    for (int d = 0; d < 5; d++) t.p[d] = lds_u32(T + 4u * ((1u << d) | (lane >> (5 - d))));
    t.s[0] = lds_u32(T + 4u * (32u + lane));
#pragma unroll
    for (int b = 0; b < 2; b++) t.s[1 + b] = lds_u32(T + 4u * (64u + 2u * lane + b));
#pragma unroll
    for (int q = 0; q < 4; q++) t.s[3 + q] = lds_u32(T + 4u * (128u + 4u * lane + q));
}
__device__ __forceinline__ void tree32_store(const Tree32& t, uint32_t T, uint32_t lane) {
#pragma unroll
    for (int d = 0; d < 5; d++) sts_u32(T + 4u * ((1u << d) | (lane >> (5 - d))), t.p[d]);
    sts_u32(T + 4u * (32u + lane), t.s[0]);
#pragma unroll
    for (int b = 0; b < 2; b++) sts_u32(T + 4u * (64u + 2u * lane + b), t.s[1 + b]);
#pragma unroll
    for (int q = 0; q < 4; q++) sts_u32(T + 4u * (128u + 4u * lane + q), t.s[3 + q]);
}
// all 8 zero-path nodes at the fixed point (lane 0 holds them all)
__device__ __forceinline__ bool tree32_zero_sat(const Tree32& t) {
    bool all = t.s[0] == kZeroSat && t.s[1] == kZeroSat && t.s[3] == kZeroSat;
#pragma unroll
    for (int d = 0; d < 5; d++) all = all && t.p[d] == kZeroSat;
    return __shfl_sync(0xFFFFFFFFu, all ? 1 : 0, 0) != 0;
}

// The coded bytes of one plane as seen by the 32 lanes of a warp that share
// one run (every lane holds the same state): a 64-bit big-endian buffer, the
// next word to append, and the word after it loaded a step ahead (a
// predicated broadcast load, so its latency is spent while other samples
// decode).  A word is appended whenever 32 bits or fewer are buffered: one
// append per sample keeps >= 32 bits buffered at a sample's start (the fast
// path checks it has the bytes it takes).  Bytes at or past the block end
// read as zero (_rc.py:129,150); loads are clamped inside the block.
struct WarpStream {
    const uint32_t* wb;  // 4-B aligned base (global)
    int32_t wend;        // bytes from wb to the block end
    int32_t wlast;       // last loadable word index (>= 0)
    uint32_t k;          // word index (from wb) of nextw
    uint32_t nextw;      // big-endian, masked
    uint32_t pend;       // raw word k + 1
    uint64_t bb;
    int32_t nbits;

    __device__ __forceinline__ const uint32_t* addr(uint32_t j) const {
        return wb + min((int32_t)j, wlast);
    }
    __device__ __forceinline__ uint32_t be_masked(uint32_t raw, uint32_t j) const {
        const int32_t vb = wend - 4 * (int32_t)j;  // valid bytes of word j
        const uint32_t m = vb >= 4 ? 0xFFFFFFFFu : (vb > 0 ? (1u << (8 * vb)) - 1u : 0u);
        return __byte_perm(raw & m, 0u, 0x0123);
    }
    __device__ __forceinline__ void init(const uint8_t* block, uint32_t len) {
        const uintptr_t st = reinterpret_cast<uintptr_t>(block) + 1;  // byte 0 is always zero
        const uintptr_t w0 = st & ~uintptr_t(3);
        const uint32_t skip = (uint32_t)(st & 3);
        wb = reinterpret_cast<const uint32_t*>(w0);
        wend = (int32_t)((reinterpret_cast<uintptr_t>(block) + len) - w0);
        wlast = max((wend - 1) >> 2, 0);
        bb = (uint64_t)(be_masked(__ldg(addr(0)), 0) << (8 * skip)) << 32;
        nbits = 32 - 8 * (int32_t)skip;
        k = 1;
        nextw = be_masked(__ldg(addr(1)), 1);
        pend = __ldg(addr(2));
        append();
    }
    __device__ __forceinline__ void append() {
        const bool need = nbits <= 32;
        const uint32_t sh = (uint32_t)(32 - nbits) & 63u;
        bb |= need ? (uint64_t)nextw << sh : 0ull;
        nbits += need ? 32 : 0;
        k += need ? 1u : 0u;
        const uint32_t nv = be_masked(pend, k);
        nextw = need ? nv : nextw;
        // the next word's load, predicated straight into `pend` (no select
        // that would wait for it)
        const uint32_t* ap = addr(k + 1);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.u32 %0, [%1];\n\t}"
                     : "+r"(pend)
                     : "l"(ap), "r"(need ? 1u : 0u));
    }
    __device__ __forceinline__ void consume(uint32_t nbytes) {  // nbytes <= 7
        bb <<= 8 * nbytes;
        nbits -= 8 * (int32_t)nbytes;
    }
    __device__ __forceinline__ uint32_t next_byte() {
        const uint32_t v = (uint32_t)(bb >> 56);
        consume(1);
        append();
        return v;
    }
};

// The careful path: the tree goes to shared memory (every lane writes the
// nodes it holds), the byte is decoded there one decision at a time exactly
// as _rc.py:136-153 (every lane redundantly: identical state, identical
// stores), and the lanes reload their nodes.
__device__ __forceinline__ uint32_t careful32(Tree32& t, uint32_t T, uint32_t lane, uint32_t& rng, uint32_t& code,
                                          WarpStream& ws) {
    tree32_store(t, T, lane);
    __syncwarp();
    atomicAdd(&g_rc_slow_bytes, 1ull);
    uint32_t ctx = 1;
    for (int k = 0; k < 8; k++) {
        const uint32_t p = lds_u32(T + 4u * ctx);
        const uint32_t bound = (rng >> 12) * p;
        const bool bit = code >= bound;
        code = bit ? code - bound : code;
        rng = bit ? rng - bound : bound;
        sts_u32(T + 4u * ctx, adapt(p, bit));
        ctx = 2 * ctx + (bit ? 1u : 0u);
        while (rng < (1u << 24)) {
            code = (code << 8) | ws.next_byte();
            rng <<= 8;
        }
    }
    __syncwarp();
    tree32_load(t, T, lane);
    return ctx & 0xFFu;
}

// Speculative evaluation of one byte on a 32-lane tree (nothing committed):
// lane i assumes the 5 leading bits i, then takes 3 decisions in its own
// subtree; the winner's interval state and a packed word (bit 31 valid, bit
// 16 a 16-bit renormalisation seen, bits 8-15 stream bytes used, bits 0-7
// the byte) reach every lane by OR-reductions (only the winner contributes).
struct Spec32 {
    uint32_t r, c, pw, pn5, pn6, pn7, b5, b6;
};
template <bool REDUX>
__device__ __forceinline__ Spec32 spec32_eval(const Tree32& t, uint32_t lane, uint32_t rng, uint32_t code,
                                              uint32_t bhi) {
    uint32_t km[5], pk[5];
#pragma unroll
    for (int d = 0; d < 5; d++) {
        km[d] = 0u - ((lane >> (4 - d)) & 1u);
        pk[d] = km[d] ? 0u - t.p[d] : t.p[d];
    }
    uint32_t a = rng >> 12, rm = rng & km[0], c = code, sel = 0x2107u, rmin = 0xFFFFFFFFu, bad = 0, rr = 0;
#pragma unroll
    for (int d = 0; d < 5; d++) kstep(a, rm, c, sel, rmin, bad, rr, t.p[d], pk[d], km[d], d < 4 ? km[d + 1] : 0u, bhi);
    Spec32 o;
    uint32_t r = rr;
    o.b5 = fstep(a, r, c, sel, rmin, o.pn5, t.s[0], bhi);
    o.b6 = fstep(a, r, c, sel, rmin, o.pn6, o.b5 ? t.s[2] : t.s[1], bhi);
    const uint32_t p7 = o.b5 ? (o.b6 ? t.s[6] : t.s[5]) : (o.b6 ? t.s[4] : t.s[3]);
    const uint32_t b7 = fstep(a, r, c, sel, rmin, o.pn7, p7, bhi);
    const bool ok = bad == 0;
    const uint32_t packed = 0x80000000u | (rmin < (1u << 16) ? 1u << 16 : 0u) | ((0x2107u - sel) << 8) |
                            (lane << 3) | (o.b5 << 2) | (o.b6 << 1) | b7;
    if (REDUX) {
        o.r = __reduce_or_sync(0xFFFFFFFFu, ok ? r : 0u);
        o.c = __reduce_or_sync(0xFFFFFFFFu, ok ? c : 0u);
        o.pw = __reduce_or_sync(0xFFFFFFFFu, ok ? packed : 0u);
    } else {  // ballot, then the winner's registers by shuffles
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
        const uint32_t w = 31u - (uint32_t)__clz(m);
        o.r = __shfl_sync(0xFFFFFFFFu, r, w);
        o.c = __shfl_sync(0xFFFFFFFFu, c, w);
        o.pw = __shfl_sync(0xFFFFFFFFu, packed, w);
        o.pw = m ? o.pw : 0u;
    }
    return o;
}
// usable without the careful path: a winner, no 16-bit shift, <= 4 bytes
__device__ __forceinline__ bool spec32_fast(uint32_t pw) {
    return (pw >> 31) != 0u && (pw & 0x10000u) == 0u && ((pw >> 8) & 0xFFu) <= 4u;
}
// adapt every lane's copies of the winner's path (branch-free): a lane holds
// the winner's depth-d node iff their top d bits agree (lane ^ w < 2^(5-d))
__device__ __forceinline__ void spec32_commit(Tree32& t, const Spec32& o, uint32_t lane) {
    const uint32_t w = (o.pw >> 3) & 31u;
    const uint32_t x = lane ^ w;
#pragma unroll
    for (int d = 0; d < 5; d++) {
        const int32_t K = ((w >> (4 - d)) & 1u) ? 15 : 4096;  // warp-uniform
        const uint32_t up = t.p[d] + (uint32_t)((K - (int32_t)t.p[d]) >> 4);
        t.p[d] = x < (32u >> d) ? up : t.p[d];
    }
    const bool iw = x == 0;
    const uint32_t q = 2u * o.b5 + o.b6;
    t.s[0] = iw ? o.pn5 : t.s[0];
    t.s[1] = (iw && !o.b5) ? o.pn6 : t.s[1];
    t.s[2] = (iw && o.b5) ? o.pn6 : t.s[2];
    t.s[3] = (iw && q == 0) ? o.pn7 : t.s[3];
    t.s[4] = (iw && q == 1) ? o.pn7 : t.s[4];
    t.s[5] = (iw && q == 2) ? o.pn7 : t.s[5];
    t.s[6] = (iw && q == 3) ? o.pn7 : t.s[6];
}
// one whole byte with its careful fallback (used off the fast path)
template <bool REDUX>
__device__ __forceinline__ uint32_t spec32_byte(Tree32& t, uint32_t T, uint32_t lane, uint32_t& rng, uint32_t& code,
                                                WarpStream& ws) {
    const Spec32 o = spec32_eval<REDUX>(t, lane, rng, code, (uint32_t)(ws.bb >> 32));
    if (!spec32_fast(o.pw)) return careful32(t, T, lane, rng, code, ws);
    spec32_commit(t, o, lane);
    rng = o.r;
    code = o.c;
    ws.consume((o.pw >> 8) & 0xFFu);
    ws.append();
    return o.pw & 0xFFu;
}

// The whole-zero-byte chain at the saturated probability: bounds b_k =
// (b_{k-1} >> 12) * 4081, valid while no renormalisation comes before the
// last decision (bp >= 2^24); the byte is zero iff code < b_8.
struct ZeroTest {
    uint32_t b, bp;
};
__device__ __forceinline__ ZeroTest zero_chain(uint32_t rng) {
    ZeroTest z;
    z.b = shr_opaque<12>(rng) * kZeroSat;
    z.bp = z.b;
#pragma unroll
    for (int k = 1; k < 8; k++) {
        z.bp = z.b;
        z.b = shr_opaque<12>(z.b) * kZeroSat;
    }
    return z;
}

// 16-bit runs: one run per warp, the tree in registers over the lanes.  Per
// sample the fast path is: the low byte by speculation, the high byte by the
// saturated zero test on the winner's state, the commit -- one branch (to the
// careful / general path) per sample.  Smem per warp: tree 0 and tree 1
// (1 KiB each, node n at +4n), used only by the careful path.
template <bool PREV, bool REDUX>
__device__ __forceinline__ void spec16_plane(Tree32& t0, Tree32& t1, bool& sat1, uint32_t T0, uint32_t T1,
                                             uint32_t lane, const PlaneRef& pr, const uint16_t* __restrict__ prev,
                                             uint16_t* __restrict__ out, uint32_t hw, uint32_t w) {
    WarpStream ws;
    ws.init(pr.coded, pr.coded_len);
    uint32_t code = (uint32_t)(ws.bb >> 32);
    ws.consume(4);
    ws.append();
    uint32_t rng = 0xFFFFFFFFu;
    uint32_t left = 0, above = 0, x = 0;
    for (uint32_t base = 0; base < hw; base += 32) {
        const uint32_t nb = min(32u, hw - base);
        uint32_t pv = 0, slot = 0;
        if (PREV && lane < nb) pv = prev[base + lane];
#pragma unroll 2
        for (uint32_t j = 0; j < nb; j++) {
            const Spec32 o = spec32_eval<REDUX>(t0, lane, rng, code, (uint32_t)(ws.bb >> 32));
            const uint32_t used = (o.pw >> 8) & 0xFFu;
            const ZeroTest zt = zero_chain(o.r);
            const uint32_t S = zt.b < (1u << 24) ? 1u : 0u;
            const uint32_t nbyte = (uint32_t)(ws.bb >> (56 - 8 * (used & 7u))) & 0xFFu;
            uint32_t z;
            if (spec32_fast(o.pw) && sat1 && zt.bp >= (1u << 24) && o.c < zt.b &&
                8 * (int32_t)(used + S) <= ws.nbits) {
                spec32_commit(t0, o, lane);
                rng = S ? zt.b << 8 : zt.b;
                code = S ? (o.c << 8) | nbyte : o.c;
                ws.consume(used + S);
                ws.append();
                z = o.pw & 0xFFu;
            } else {  // rare: the careful low byte and/or the general high byte
                uint32_t lo;
                if (!spec32_fast(o.pw) || 8 * (int32_t)used > ws.nbits) {
                    lo = careful32(t0, T0, lane, rng, code, ws);
                } else {
                    spec32_commit(t0, o, lane);
                    rng = o.r;
                    code = o.c;
                    ws.consume(used);
                    ws.append();
                    ws.append();
                    lo = o.pw & 0xFFu;
                }
                const ZeroTest z2 = zero_chain(rng);
                uint32_t hi = 0;
                if (sat1 && z2.bp >= (1u << 24) && code < z2.b) {
                    const uint32_t S2 = z2.b < (1u << 24) ? 1u : 0u;
                    rng = S2 ? z2.b << 8 : z2.b;
                    code = S2 ? (code << 8) | (uint32_t)(ws.bb >> 56) : code;
                    ws.consume(S2);
                    ws.append();
                } else {
                    hi = spec32_byte<REDUX>(t1, T1, lane, rng, code, ws);
                    sat1 = tree32_zero_sat(t1);
                }
                z = lo | hi << 8;
            }
            const uint32_t r = (z >> 1) ^ (0u - (z & 1u));
            if (PREV) {
                slot = lane == j ? r : slot;
            } else {
                const uint32_t idx = base + j;
                const uint32_t pred = x > 0 ? left : (idx > 0 ? above : 0x8000u);
                const uint32_t v = (pred + r) & 0xFFFFu;
                above = x == 0 ? v : above;
                left = v;
                x = x + 1 == w ? 0u : x + 1;
                slot = lane == j ? v : slot;
            }
        }
        if (lane < nb) out[base + lane] = (uint16_t)(PREV ? pv + slot : slot);
    }
}

template <bool REDUX>
__device__ __forceinline__ void spec16_run(const RunDesc& r, const PlaneRef* __restrict__ planes, uint32_t T0,
                                           uint32_t T1, uint32_t lane) {
    Tree32 t0, t1;
#pragma unroll
    for (int d = 0; d < 5; d++) {  // new_bittree_probs (_rc.py:304-317): zero-path nodes 3686
        t0.p[d] = t1.p[d] = (lane >> (5 - d)) == 0 ? 3686u : 2048u;
    }
#pragma unroll
    for (int k = 0; k < 7; k++) t0.s[k] = t1.s[k] = 2048u;
    if (lane == 0) t0.s[0] = t0.s[1] = t0.s[3] = t1.s[0] = t1.s[1] = t1.s[3] = 3686u;
    bool sat1 = false;
    const uint32_t hw = (uint32_t)r.w * r.h;
    for (int f = 0; f < r.count; f++) {
        const PlaneRef pr = planes[r.plane_base + f];
        if (pr.mode != 0) continue;  // RAW plane (already copied to aligned storage)
        uint16_t* out = reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(pr.samples));
        if (f > 0)
            spec16_plane<true, REDUX>(t0, t1, sat1, T0, T1, lane, pr,
                               reinterpret_cast<const uint16_t*>(planes[r.plane_base + f - 1].samples), out, hw, r.w);
        else
            spec16_plane<false, REDUX>(t0, t1, sat1, T0, T1, lane, pr, nullptr, out, hw, r.w);
    }
}

// One tree over the 16 lanes h of a half warp, 8-bit runs: q[d] = node
// (16 << d) | (h >> (4 - d)) (the low nibble's nodes on the lane's path; the
// zero-path nodes 1, 2, 4, 8 sit at 4081 whenever the fast path runs).
struct Tree16 {
    uint32_t q[4];
};
__device__ __forceinline__ void tree16_load(Tree16& t, uint32_t T, uint32_t h) {
#pragma unroll
    for (int d = 0; d < 4; d++) t.q[d] = lds_u32(T + 4u * ((16u << d) | (h >> (4 - d))));
}
__device__ __forceinline__ bool tree16_sat(uint32_t T) {
    return lds_u32(T + 4u) == kZeroSat && lds_u32(T + 8u) == kZeroSat && lds_u32(T + 16u) == kZeroSat &&
           lds_u32(T + 32u) == kZeroSat;
}

__device__ __forceinline__ uint32_t careful16(Tree16& t, uint32_t T, uint32_t h, uint32_t hmask, uint32_t& rng,
                                          uint32_t& code, CodedStream& cs, bool& sat) {
#pragma unroll
    for (int d = 0; d < 4; d++) sts_u32(T + 4u * ((16u << d) | (h >> (4 - d))), t.q[d]);
    __syncwarp(hmask);
    uint4 q0 = lds_quad(T);
    const uint32_t v = decode_byte_slow(T, T, q0, rng, code, cs);
    __syncwarp(hmask);
    tree16_load(t, T, h);
    sat = tree16_sat(T);
    return v;
}

__device__ __forceinline__ uint32_t spec_byte16(Tree16& t, uint32_t T, uint32_t h, uint32_t hmask, uint32_t& rng,
                                                uint32_t& code, CodedStream& cs, bool& sat) {
    if (!sat) return careful16(t, T, h, hmask, rng, code, cs, sat);
    const uint32_t bhi = (uint32_t)(cs.bb >> 32);
    uint32_t km[4], pk[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        km[d] = 0u - ((h >> (3 - d)) & 1u);
        pk[d] = km[d] ? 0u - t.q[d] : t.q[d];
    }
    uint32_t a = rng >> 12, r = rng, c = code, sel = 0x2107u, rmin = 0xFFFFFFFFu, bad = 0, rr = 0;
#pragma unroll
    for (int d = 0; d < 4; d++) zstep(a, r, c, sel, rmin, bad, bhi);
    uint32_t rm = r & km[0];
#pragma unroll
    for (int d = 0; d < 4; d++) kstep(a, rm, c, sel, rmin, bad, rr, t.q[d], pk[d], km[d], d < 3 ? km[d + 1] : 0u, bhi);
    const uint32_t shift = (threadIdx.x & 16u);
    const uint32_t m = (__ballot_sync(hmask, bad == 0) >> shift) & 0xFFFFu;
    const uint32_t w = __ffs(m) - 1;
    const uint32_t packed = h | ((0x2107u - sel) << 8) | (rmin < (1u << 16) ? 1u << 16 : 0u);
    const uint32_t src = (w & 15u) | shift;
    const uint32_t nr = __shfl_sync(hmask, rr, src);
    const uint32_t nc = __shfl_sync(hmask, c, src);
    const uint32_t pw = __shfl_sync(hmask, packed, src);
    const uint32_t used = (pw >> 8) & 0xFFu;
    if (m == 0 || (pw >> 16) != 0 || used > 4u) return careful16(t, T, h, hmask, rng, code, cs, sat);
    rng = nr;
    code = nc;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const bool match = ((h ^ w) >> (4 - d)) == 0;
        if (match) t.q[d] = adapt_u(t.q[d], (w >> (3 - d)) & 1u);
    }
    cs.bb <<= 8 * used;
    cs.nbits -= (int32_t)(8 * used);
    cs.refill();
    return pw & 0xFu;
}

template <bool PREV>
__device__ __forceinline__ void spec8_plane(Tree16& t, bool& sat, uint32_t T, uint32_t R, uint32_t h,
                                            uint32_t hmask, const PlaneRef& pr, const uint8_t* __restrict__ prev,
                                            uint8_t* __restrict__ out, uint32_t hw, uint32_t w) {
    CodedStream cs;
    cs.init(pr.coded, pr.coded_len, R);
    uint32_t code = cs.take32();
    cs.refill();
    uint32_t rng = 0xFFFFFFFFu;
    uint32_t left = 0, above = 0, x = 0;
    for (uint32_t base = 0; base < hw; base += 16) {
        const uint32_t nb = min(16u, hw - base);
        uint32_t pv = 0, slot = 0;
        if (PREV && h < nb) pv = prev[base + h];
#pragma unroll 1
        for (uint32_t j = 0; j < nb; j++) {
            const uint32_t z = spec_byte16(t, T, h, hmask, rng, code, cs, sat);
            const uint32_t r = (z >> 1) ^ (0u - (z & 1u));
            if (PREV) {
                if (h == j) slot = r;
            } else {
                const uint32_t idx = base + j;
                const uint32_t pred = x > 0 ? left : (idx > 0 ? above : 0x80u);
                const uint32_t v = (pred + r) & 0xFFu;
                if (x == 0) above = v;
                left = v;
                if (++x == w) x = 0;
                if (h == j) slot = v;
            }
        }
        if (h < nb) out[base + h] = (uint8_t)(PREV ? pv + slot : slot);
    }
    cs.finish();
}

__device__ __forceinline__ void spec8_run(const RunDesc& r, const PlaneRef* __restrict__ planes, uint32_t T,
                                          uint32_t R, uint32_t h, uint32_t hmask) {
    // new_bittree_probs (_rc.py:304-317): the whole tree in shared memory
    // (the careful path's home), the lane copies loaded from it
    for (uint32_t i = h; i < 256; i += 16) sts_u32(T + 4u * i, (i != 0 && (i & (i - 1)) == 0) ? 3686u : 2048u);
    __syncwarp(hmask);
    Tree16 t;
    tree16_load(t, T, h);
    bool sat = false;
    const uint32_t hw = (uint32_t)r.w * r.h;
    for (int f = 0; f < r.count; f++) {
        const PlaneRef pr = planes[r.plane_base + f];
        if (pr.mode != 0) continue;
        uint8_t* out = const_cast<uint8_t*>(pr.samples);
        if (f > 0)
            spec8_plane<true>(t, sat, T, R, h, hmask, pr, planes[r.plane_base + f - 1].samples, out, hw, r.w);
        else
            spec8_plane<false>(t, sat, T, R, h, hmask, pr, nullptr, out, hw, r.w);
    }
}

// ---------------------------------------------------------------------------
// 8-bit runs, a lane per run (32 runs per warp in lock-step), branch-light:
// the low-nibble subtree (15 nodes: 16, 32-33, 64-67, 128-135) lives in the
// lane's REGISTERS; while the zero-path nodes 1, 2, 4, 8 sit at the fixed
// point 4081 (8-bit residuals here never leave the low nibble) a byte is 4
// zero decisions at p = 4081 + 4 decisions on the register subtree, the
// probability of each taken from registers by selects prepared one decision
// ahead, and the commit writes the 4 adapted nodes back by selects.  Any
// other byte (a 1 in the top nibble, a 16-bit renormalisation, > 4 stream
// bytes, the zero path not yet saturated) goes to the careful path on the
// lane's shared-memory tree (the subtree is written there first and reloaded
// after).  The stream is the WarpStream scheme per lane (the next word's
// load predicated a step ahead).
struct LaneStream {
    const uint32_t* wb;
    int32_t wend, wlast;
    uint32_t k, nextw, pend;
    uint64_t bb;
    int32_t nbits;
    __device__ __forceinline__ const uint32_t* addr(uint32_t j) const { return wb + min((int32_t)j, wlast); }
    __device__ __forceinline__ uint32_t be_masked(uint32_t raw, uint32_t j) const {
        const int32_t vb = wend - 4 * (int32_t)j;
        const uint32_t m = vb >= 4 ? 0xFFFFFFFFu : (vb > 0 ? (1u << (8 * vb)) - 1u : 0u);
        return __byte_perm(raw & m, 0u, 0x0123);
    }
    __device__ __forceinline__ void init(const uint8_t* block, uint32_t len) {
        const uintptr_t st = reinterpret_cast<uintptr_t>(block) + 1;
        const uintptr_t w0 = st & ~uintptr_t(3);
        const uint32_t skip = (uint32_t)(st & 3);
        wb = reinterpret_cast<const uint32_t*>(w0);
        wend = (int32_t)((reinterpret_cast<uintptr_t>(block) + len) - w0);
        wlast = max((wend - 1) >> 2, 0);
        bb = (uint64_t)(be_masked(__ldg(addr(0)), 0) << (8 * skip)) << 32;
        nbits = 32 - 8 * (int32_t)skip;
        k = 1;
        nextw = be_masked(__ldg(addr(1)), 1);
        pend = __ldg(addr(2));
        append();
    }
    __device__ __forceinline__ void append() {
        const bool need = nbits <= 32;
        const uint32_t sh = (uint32_t)(32 - nbits) & 63u;
        bb |= need ? (uint64_t)nextw << sh : 0ull;
        nbits += need ? 32 : 0;
        k += need ? 1u : 0u;
        const uint32_t nv = be_masked(pend, k);
        nextw = need ? nv : nextw;
        const uint32_t* ap = addr(k + 1);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.u32 %0, [%1];\n\t}"
                     : "+r"(pend)
                     : "l"(ap), "r"(need ? 1u : 0u));
    }
    __device__ __forceinline__ void consume(uint32_t nbytes) {
        bb <<= 8 * nbytes;
        nbits -= 8 * (int32_t)nbytes;
    }
    __device__ __forceinline__ uint32_t next_byte() {
        const uint32_t v = (uint32_t)(bb >> 56);
        consume(1);
        append();
        return v;
    }
};

// subtree register index of node (16 << j) + q is (1 << j) - 1 + q
__device__ __forceinline__ uint32_t nib_node(int i) {
    return i == 0 ? 16u : (i < 3 ? 32u + (i - 1) : (i < 7 ? 64u + (i - 3) : 128u + (i - 7)));
}

__device__ __forceinline__ uint32_t lane8_careful(uint32_t (&n)[15], uint32_t T, uint32_t& rng, uint32_t& code,
                                                  LaneStream& ls, bool& sat) {
#pragma unroll
    for (int i = 0; i < 15; i++) sts_u32(T + 4u * nib_node(i), n[i]);
    atomicAdd(&g_rc_slow_bytes, 1ull);
    uint32_t ctx = 1;
    for (int k = 0; k < 8; k++) {
        const uint32_t p = lds_u32(T + 4u * ctx);
        const uint32_t bound = (rng >> 12) * p;
        const bool bit = code >= bound;
        code = bit ? code - bound : code;
        rng = bit ? rng - bound : bound;
        sts_u32(T + 4u * ctx, adapt(p, bit));
        ctx = 2 * ctx + (bit ? 1u : 0u);
        while (rng < (1u << 24)) {
            code = (code << 8) | ls.next_byte();
            rng <<= 8;
        }
    }
#pragma unroll
    for (int i = 0; i < 15; i++) n[i] = lds_u32(T + 4u * nib_node(i));
    sat = lds_u32(T + 4u) == kZeroSat && lds_u32(T + 8u) == kZeroSat && lds_u32(T + 16u) == kZeroSat &&
          lds_u32(T + 32u) == kZeroSat;
    return ctx & 0xFFu;
}

template <bool PREV>
__device__ __forceinline__ void lane8_plane(uint32_t (&n)[15], bool& sat, uint32_t T, const PlaneRef& pr,
                                            const uint32_t* __restrict__ prev, uint32_t* __restrict__ out,
                                            uint32_t hw, uint32_t w) {
    LaneStream ls;
    ls.init(pr.coded, pr.coded_len);
    uint32_t code = (uint32_t)(ls.bb >> 32);
    ls.consume(4);
    ls.append();
    uint32_t rng = 0xFFFFFFFFu;
    uint32_t left = 0, above = 0, x = 0;
    auto sample = [&](uint32_t idx, uint32_t pw, uint32_t j) -> uint32_t {
            const uint32_t bhi = (uint32_t)(ls.bb >> 32);
            uint32_t a = rng >> 12, r = rng, c = code, sel = 0x2107u, rmin = 0xFFFFFFFFu, bad = 0;
#pragma unroll
            for (int d = 0; d < 4; d++) zstep(a, r, c, sel, rmin, bad, bhi);
            uint32_t pn4, pn5, pn6, pn7;
            const uint32_t b4 = fstep(a, r, c, sel, rmin, pn4, n[0], bhi);
            const uint32_t x0 = b4 ? n[5] : n[3], x1 = b4 ? n[6] : n[4];
            const uint32_t y00 = b4 ? n[11] : n[7], y01 = b4 ? n[12] : n[8];
            const uint32_t y10 = b4 ? n[13] : n[9], y11 = b4 ? n[14] : n[10];
            const uint32_t b5 = fstep(a, r, c, sel, rmin, pn5, b4 ? n[2] : n[1], bhi);
            const uint32_t y0 = b5 ? y10 : y00, y1 = b5 ? y11 : y01;
            const uint32_t b6 = fstep(a, r, c, sel, rmin, pn6, b5 ? x1 : x0, bhi);
            const uint32_t b7 = fstep(a, r, c, sel, rmin, pn7, b6 ? y1 : y0, bhi);
            const uint32_t used = 0x2107u - sel;
            uint32_t z;
            if (sat && bad == 0 && rmin >= (1u << 16) && used <= 4u && 8 * (int32_t)used <= ls.nbits) {
                n[0] = pn4;
                n[1] = b4 ? n[1] : pn5;
                n[2] = b4 ? pn5 : n[2];
                const uint32_t i6 = 2u * b4 + b5;
#pragma unroll
                for (int q = 0; q < 4; q++) n[3 + q] = i6 == (uint32_t)q ? pn6 : n[3 + q];
                const uint32_t i7 = 4u * b4 + 2u * b5 + b6;
#pragma unroll
                for (int q = 0; q < 8; q++) n[7 + q] = i7 == (uint32_t)q ? pn7 : n[7 + q];
                rng = r;
                code = c;
                ls.consume(used);
                ls.append();
                z = (b4 << 3) | (b5 << 2) | (b6 << 1) | b7;
            } else {
                z = lane8_careful(n, T, rng, code, ls, sat);
            }
            const uint32_t rr = (z >> 1) ^ (0u - (z & 1u));
            uint32_t v;
            if (PREV) {
                v = ((pw >> (8 * j)) + rr) & 0xFFu;
            } else {
                const uint32_t pred = x > 0 ? left : (idx > 0 ? above : 0x80u);
                v = (pred + rr) & 0xFFu;
                above = x == 0 ? v : above;
                left = v;
                x = x + 1 == w ? 0u : x + 1;
            }
            return v << (8 * j);
    };
    const uint32_t full = hw / 4;
    for (uint32_t wi = 0; wi < full; wi++) {  // 4 samples per word, unrolled
        const uint32_t pw = PREV ? __ldg(prev + wi) : 0u;
        uint32_t ow = 0;
#pragma unroll
        for (uint32_t j = 0; j < 4; j++) ow |= sample(4 * wi + j, pw, j);
        out[wi] = ow;
    }
    if (hw & 3u) {
        const uint32_t pw = PREV ? __ldg(prev + full) : 0u;
        uint32_t ow = 0;
        for (uint32_t j = 0; j < (hw & 3u); j++) ow |= sample(4 * full + j, pw, j);
        out[full] = ow;
    }
}

__device__ __forceinline__ void lane8_run(const RunDesc& r, const PlaneRef* __restrict__ planes, uint32_t T) {
    for (uint32_t i = 0; i < 256; i++) sts_u32(T + 4u * i, (i != 0 && (i & (i - 1)) == 0) ? 3686u : 2048u);
    uint32_t n[15];
#pragma unroll
    for (int i = 0; i < 15; i++) n[i] = lds_u32(T + 4u * nib_node(i));
    bool sat = false;
    const uint32_t hw = (uint32_t)r.w * r.h;
    for (int f = 0; f < r.count; f++) {
        const PlaneRef pr = planes[r.plane_base + f];
        if (pr.mode != 0) continue;
        uint32_t* out = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(pr.samples));
        if (f > 0)
            lane8_plane<true>(n, sat, T, pr, reinterpret_cast<const uint32_t*>(planes[r.plane_base + f - 1].samples),
                              out, hw, r.w);
        else
            lane8_plane<false>(n, sat, T, pr, nullptr, out, hw, r.w);
    }
}

constexpr uint32_t kSpecSmem = 2 * (kRingBytes + kTreeBytes);  // per block (2 u8 runs, or 1 u16 run with 2 trees)

// One launch for every width class (no serialisation of the u8 and u16 runs
// behind each other): blocks [0, nb1) decode the 8-bit runs, the next nb2
// blocks the 16-bit runs, the rest the 32-bit runs.  One warp per CTA, so
// the warps land on separate SMs.
template <int V, int NB>
__device__ __forceinline__ void decode_runs(const RunDesc* __restrict__ runs, const uint32_t* __restrict__ rc_runs,
                                            int n, int blk, const PlaneRef* __restrict__ planes, uint32_t P,
                                            uint32_t R, int prof_base) {
    const int lane = threadIdx.x;
    for (int b = 0; b < NB; b++)  // new_bittree_probs (_rc.py:304-317)
        for (uint32_t i = 0; i < 256; i++)
            sts_u32(node_addr(P + b * kTreeBytes, i), (i != 0 && (i & (i - 1)) == 0) ? 3686u : 2048u);
    const int gi = blk * (int)blockDim.x + lane;
    if (gi >= n) return;
    const long long t0 = clock64();
    const RunDesc r = runs[rc_runs[gi]];
    const uint32_t hw = (uint32_t)r.w * r.h;
    bool sat = false;  // variant 4: zero-path probabilities saturated (persists with the model)
    for (int f = 0; f < r.count; f++) {
        const PlaneRef pr = planes[r.plane_base + f];
        if (pr.mode != 0) continue;  // RAW plane (already copied to aligned storage)
        uint32_t* out = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(pr.samples));
        if (f > 0) {
            const uint32_t* prev = reinterpret_cast<const uint32_t*>(planes[r.plane_base + f - 1].samples);
            decode_plane<V, NB, true>(P, R, pr, prev, out, hw, r.w, sat);
        } else {
            decode_plane<V, NB, false>(P, R, pr, nullptr, out, hw, r.w, sat);
        }
    }
    if (unsigned long long* prof = g_rc_prof) {
        prof[2 * (prof_base + gi)] = rc_runs[gi];
        prof[2 * (prof_base + gi) + 1] = (unsigned long long)(clock64() - t0);
    }
}

struct RcClasses {
    int n[3];    // runs per class (1, 2, 4 bytes per sample)
    int off[3];  // first index into rc_runs
    int blk[4];  // block prefix
    int u8_spec; // variant 5: 8-bit runs by half-warp speculation (else a lane per run)
    int skip;    // dev isolation probe: bit k skips class k (results wrong by design)
};

template <int V>
__global__ void __launch_bounds__(32) rc_decode_kernel(const RunDesc* __restrict__ runs,
                                                         const uint32_t* __restrict__ rc_runs, RcClasses c,
                                                         const PlaneRef* __restrict__ planes) {
    extern __shared__ uint4 probs_s[];
    const int b = blockIdx.x;
    if (V >= 5 && (c.skip >> (b < c.blk[1] ? 0 : (b < c.blk[2] ? 1 : 2)) & 1)) return;
    if (V >= 5 && b < c.blk[2] && (c.u8_spec == 1 || b >= c.blk[1])) {
        // variant 5: blocks [0, blk1): two 8-bit runs each; [blk1, blk2): one 16-bit run each
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(probs_s);
        const uint32_t lane = threadIdx.x;
        const long long t0 = clock64();
        int gi;
        if (b < c.blk[1]) {
            const uint32_t half = lane >> 4, h = lane & 15u, hmask = 0xFFFFu << (16 * half);
            gi = 2 * b + (int)half;
            if (gi >= c.n[0]) return;
            const uint32_t R = base + half * (kRingBytes + kTreeBytes);
            spec8_run(runs[rc_runs[c.off[0] + gi]], planes, R + kRingBytes, R, h, hmask);
            gi += c.off[0];
            if (h != 0) return;
        } else {
            gi = b - c.blk[1];
            spec16_run<V == 5>(runs[rc_runs[c.off[1] + gi]], planes, base + kRingBytes, base + kRingBytes + kTreeBytes,
                               lane);
            gi += c.off[1];
            if (lane != 0) return;
        }
        if (unsigned long long* prof = g_rc_prof) {
            prof[2 * gi] = rc_runs[gi];
            prof[2 * gi + 1] = (unsigned long long)(clock64() - t0);
        }
        return;
    }
    const int nb = b < c.blk[1] ? 1 : (b < c.blk[2] ? 2 : 4);
    if constexpr (V >= 5) {  // 32-bit (and lane-per-run 8-bit) runs: variant 4
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(probs_s);
        const uint32_t R = base + threadIdx.x * kRingBytes;
        const uint32_t P = base + blockDim.x * kRingBytes + threadIdx.x * lane_stride(nb);
        if (b < c.blk[1] && c.u8_spec == 2) {
            const int gi = b * 32 + (int)threadIdx.x;
            if (gi >= c.n[0]) return;
            const long long t0 = clock64();
            lane8_run(runs[rc_runs[c.off[0] + gi]], planes, base + threadIdx.x * (kTreeBytes + 16u));
            if (unsigned long long* prof = g_rc_prof) {
                prof[2 * (c.off[0] + gi)] = rc_runs[c.off[0] + gi];
                prof[2 * (c.off[0] + gi) + 1] = (unsigned long long)(clock64() - t0);
            }
        } else if (b < c.blk[1]) decode_runs<4, 1>(runs, rc_runs + c.off[0], c.n[0], b, planes, P, R, c.off[0]);
        else decode_runs<4, 4>(runs, rc_runs + c.off[2], c.n[2], b - c.blk[2], planes, P, R, c.off[2]);
    } else {
    // lane rings of coded bytes first, then the lane-private probability trees
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(probs_s);
    const uint32_t R = base + threadIdx.x * kRingBytes;
    const uint32_t P = base + blockDim.x * kRingBytes + threadIdx.x * lane_stride(nb);
    if (b < c.blk[1]) decode_runs<V, 1>(runs, rc_runs + c.off[0], c.n[0], b, planes, P, R, c.off[0]);
    else if (b < c.blk[2])
        decode_runs<V, 2>(runs, rc_runs + c.off[1], c.n[1], b - c.blk[1], planes, P, R, c.off[1]);
    else decode_runs<V, 4>(runs, rc_runs + c.off[2], c.n[2], b - c.blk[2], planes, P, R, c.off[2]);
    }
}

void launch_rc_decode(const RunDesc* runs, const uint32_t* rc_runs, const int* n_per_class,
                      const PlaneRef* planes, cudaStream_t s) {
    RcClasses c;
    int nbmax = 0, off = 0;
    const char* er = getenv("GSV_RC_RPW");  // runs per warp (dev tuning)
    int rpw = er ? atoi(er) : kRPW;
    rpw = rpw < 1 ? 1 : (rpw > 32 ? 32 : rpw);
    const char* ev = getenv("GSV_RC_VARIANT");  // decoder variant (dev tuning)
    const int v = ev ? atoi(ev) : 6;
    const char* e8 = getenv("GSV_RC_U8_SPEC");
    c.u8_spec = e8 ? atoi(e8) : 2;
    const char* es = getenv("GSV_RC_SKIP");
    c.skip = es ? atoi(es) : 0;
    c.blk[0] = 0;
    for (int k = 0; k < 3; k++) {
        c.n[k] = n_per_class[k];
        c.off[k] = off;
        off += c.n[k];
        // variant 5: 2 runs per block (8-bit), 1 (16-bit); 32-bit runs rpw per block
        const int per = v >= 5 ? (k == 0 ? (c.u8_spec == 1 ? 2 : 32) : (k == 1 ? 1 : 32)) : rpw;
        c.blk[k + 1] = c.blk[k] + (c.n[k] + per - 1) / per;
        if (c.n[k] > 0) nbmax = 1 << k;
    }
    if (c.blk[3] == 0) return;
    size_t smem = (size_t)(lane_stride(nbmax) + kRingBytes) * rpw;
    if (v >= 5) {
        smem = kSpecSmem;
        if (c.n[0] > 0 && c.u8_spec != 1) smem = std::max(smem, (size_t)(lane_stride(1) + kRingBytes) * 32);
        if (c.n[2] > 0) smem = std::max(smem, (size_t)(lane_stride(4) + kRingBytes) * 32);
        if (v == 6) {
            cudaFuncSetAttribute(rc_decode_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            rc_decode_kernel<6><<<c.blk[3], 32, smem, s>>>(runs, rc_runs, c, planes);
        } else {
            cudaFuncSetAttribute(rc_decode_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            rc_decode_kernel<5><<<c.blk[3], 32, smem, s>>>(runs, rc_runs, c, planes);
        }
    } else if (v == 4) {
        cudaFuncSetAttribute(rc_decode_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rc_decode_kernel<4><<<c.blk[3], rpw, smem, s>>>(runs, rc_runs, c, planes);
    } else if (v == 3) {
        cudaFuncSetAttribute(rc_decode_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rc_decode_kernel<3><<<c.blk[3], rpw, smem, s>>>(runs, rc_runs, c, planes);
    } else if (v == 1) {
        cudaFuncSetAttribute(rc_decode_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rc_decode_kernel<1><<<c.blk[3], rpw, smem, s>>>(runs, rc_runs, c, planes);
    } else {
        cudaFuncSetAttribute(rc_decode_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rc_decode_kernel<2><<<c.blk[3], rpw, smem, s>>>(runs, rc_runs, c, planes);
    }
}

}  // namespace gsv

// dev: per-run decode cycles into `buf` (2 x u64 per range-coded run), or off
extern "C" int gsv_dev_rc_profile(unsigned long long* buf) {
    return cudaMemcpyToSymbol(gsv::g_rc_prof, &buf, sizeof buf) == cudaSuccess ? 0 : -1;
}

extern "C" unsigned long long gsv_dev_rc_slow_bytes(int reset) {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, gsv::g_rc_slow_bytes, sizeof v);
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(gsv::g_rc_slow_bytes, &z, sizeof z);
    }
    return v;
}
