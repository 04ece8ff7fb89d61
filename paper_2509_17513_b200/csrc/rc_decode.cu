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
//     reading the previous plane and writing the output as aligned words.
// RAW-mode planes of these runs are first copied to 16-B aligned storage so
// that every predictor plane is aligned.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

constexpr int kRPW = 32;  // runs per warp

__global__ void copy_planes_kernel(const CopyJob* __restrict__ jobs, int njobs) {
    for (int j = blockIdx.x; j < njobs; j += gridDim.x) {
        const CopyJob cj = jobs[j];
        for (uint32_t i = threadIdx.x; i < cj.bytes; i += blockDim.x) cj.dst[i] = __ldg(cj.src + i);
    }
}

void launch_copy_planes(const CopyJob* jobs, int njobs, cudaStream_t s) {
    if (njobs <= 0) return;
    copy_planes_kernel<<<min(njobs, 148 * 8), 256, 0, s>>>(jobs, njobs);
}

// Coded bytes as a big-endian bit buffer: the next byte sits in bits 63..56
// of `bb`, so a renormalisation by `sh` (0, 8 or 16) bits is one funnel
// shift into `code` plus a 64-bit shift of `bb`.  `bb` is refilled 32 bits
// at a time from a 4-word register queue of aligned loads issued ~16 bytes
// ahead.  Bytes past the block read as zero (_rc.py:129,150).
struct CodedStream {
    const uint32_t* wp;  // next aligned word to load
    uint32_t r0, r1, r2, r3;
    uint64_t bb;
    int32_t nbits;       // valid bits in bb
    int32_t left;        // stream bytes not yet moved into bb (<= 0: zero fill)

    __device__ __forceinline__ uint32_t pop() {
        const uint32_t w = r0;
        r0 = r1;
        r1 = r2;
        r2 = r3;
        r3 = __ldg(wp++);
        return w;
    }
    // big-endian word with only its first m bytes kept
    __device__ __forceinline__ static uint32_t be_keep(uint32_t w_le, int32_t m) {
        const uint32_t be = __byte_perm(w_le, 0u, 0x0123);
        return m >= 4 ? be : (m > 0 ? be & ~(0xFFFFFFFFu >> (8 * m)) : 0u);
    }
    __device__ __forceinline__ void init(const uint8_t* block, uint32_t len) {
        const uintptr_t s = reinterpret_cast<uintptr_t>(block) + 1;  // byte 0 is always zero
        wp = reinterpret_cast<const uint32_t*>(s & ~uintptr_t(3));
        const int k = (int)(s & 3);
        r0 = __ldg(wp);
        r1 = __ldg(wp + 1);
        r2 = __ldg(wp + 2);
        r3 = __ldg(wp + 3);
        wp += 4;
        left = (int32_t)len - 1;
        const int nb = 4 - k;
        const uint32_t be = __byte_perm(pop(), 0u, 0x0123) << (8 * k);  // first nb bytes on top
        const int32_t m = left < nb ? left : nb;
        const uint32_t kept = m >= 4 ? be : (m > 0 ? be & ~(0xFFFFFFFFu >> (8 * m)) : 0u);
        left -= nb;
        bb = (uint64_t)kept << 32;
        nbits = 8 * nb;
        refill();
    }
    __device__ __forceinline__ void refill() {
        if (nbits <= 32) {
            const uint32_t w = be_keep(pop(), left);
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

// Fast path: the byte's decisions read the coded bits at a running offset
// into the 64-bit buffer (one funnel shift) and defer the 8 probability
// stores to the end of the byte, so a decision is: multiply, compare, select,
// renormalise -- no buffer bookkeeping, no store, no branch.  It is exact as
// long as the byte consumes at most 32 bits (>= 33 are buffered at the start);
// otherwise nothing has been written and the byte is redone on the careful
// path from the saved state.  Multi-byte samples alternate trees, so q0 of
// the next tree is loaded during this byte; for one-byte samples the next
// root quad is this tree's, patched in registers with the new node 1..3.
template <bool SAME_TREE>
__device__ __forceinline__ uint32_t decode_byte(uint32_t T, uint32_t Tn, uint4& q0, uint32_t& rng,
                                                uint32_t& code, CodedStream& cs) {
    const uint32_t rng0 = rng, code0 = code;
    const uint32_t bhi = (uint32_t)(cs.bb >> 32), blo = (uint32_t)cs.bb;
    uint32_t ctx = 1, off = 0;
    uint32_t p = q0.y;
    uint4 cq = q0;
    uint4 qn = q0;
    uint32_t pn[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint4 nq = make_uint4(0u, 0u, 0u, 0u);
        if (k < 6) nq = lds_quad(T + ctx * 16u);
        if (!SAME_TREE && k == 6) qn = lds_quad(Tn);
        const uint32_t c0 = (ctx & 1) ? cq.z : cq.x;
        const uint32_t c1 = (ctx & 1) ? cq.w : cq.y;
        const uint32_t bound = (rng >> 12) * p;
        const bool bit = code >= bound;
        code = bit ? code - bound : code;
        rng = bit ? rng - bound : bound;
        pn[k] = adapt(p, bit);
        ctx = 2 * ctx + (bit ? 1u : 0u);
        p = bit ? c1 : c0;
        cq = nq;
        const uint32_t sh = rng < (1u << 24) ? (rng < (1u << 16) ? 16u : 8u) : 0u;
        code = __funnelshift_l(__funnelshift_lc(blo, bhi, off), code, sh);
        rng <<= sh;
        off += sh;
    }
    if (off > 32u) {  // rare: redo carefully (nothing was stored)
        rng = rng0;
        code = code0;
        return decode_byte_slow(T, Tn, q0, rng, code, cs);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) sts_u32(node_addr(T, ctx >> (8 - k)), pn[k]);
    if (SAME_TREE) {
        const bool b0 = (ctx >> 7) & 1u;  // first decision: node 2 or 3 was updated second
        qn.y = pn[0];
        qn.z = b0 ? q0.z : pn[1];
        qn.w = b0 ? pn[1] : q0.w;
    }
    q0 = qn;
    cs.bb <<= off;
    cs.nbits -= (int32_t)off;
    cs.refill();
    return ctx & 0xFFu;
}

template <int NB, bool PREV>
__device__ __forceinline__ void decode_plane(uint32_t P, const PlaneRef& pr,
                                             const uint32_t* __restrict__ prev,
                                             uint32_t* __restrict__ out, uint32_t hw, uint32_t w) {
    constexpr int SPW = 4 / NB;  // samples per 32-bit word
    constexpr uint32_t mask = NB == 4 ? 0xFFFFFFFFu : ((1u << (8 * NB)) - 1u);
    constexpr uint32_t def = 128u << (8 * NB - 8);
    CodedStream cs;
    cs.init(pr.coded, pr.coded_len);
    uint32_t code = cs.take32();
    cs.refill();
    uint32_t rng = 0xFFFFFFFFu;
    uint4 q0 = lds_quad(P);                  // root quad of tree 0
    uint32_t pq0 = 0, pq1 = 0, pq2 = 0, pq3 = 0;  // previous-plane word queue
    const uint32_t* pp = prev;
    if (PREV) {
        pq0 = pp[0];
        pq1 = pp[1];
        pq2 = pp[2];
        pq3 = pp[3];
        pp += 4;
    }
    uint32_t left = 0, above = 0, x = 0;
    const uint32_t nwords = (hw * NB + 3) / 4;
    uint32_t idx = 0;
    for (uint32_t wi = 0; wi < nwords; wi++) {
        uint32_t pw = 0;
        if (PREV) {
            pw = pq0;
            pq0 = pq1;
            pq1 = pq2;
            pq2 = pq3;
            pq3 = pp[0];
            pp++;
        }
        uint32_t ow = 0;
#pragma unroll
        for (int j = 0; j < SPW; j++) {
            if (SPW > 1 && idx >= hw) break;
            uint32_t pred;
            if (PREV) {
                pred = (pw >> (8 * NB * j)) & mask;
            } else {
                pred = x > 0 ? left : (idx > 0 ? above : def);
            }
            uint32_t z = 0;
#pragma unroll
            for (int b = 0; b < NB; b++)
                z |= decode_byte<NB == 1>(P + b * kTreeBytes, P + ((b + 1) % NB) * kTreeBytes, q0, rng,
                                          code, cs) << (8 * b);
            const uint32_t v = (pred + ((z >> 1) ^ (0u - (z & 1u)))) & mask;  // unzigzag
            if (!PREV) {
                if (x == 0) above = v;
                left = v;
                if (++x == w) x = 0;
            }
            ow |= v << (8 * NB * j);
            idx++;
        }
        out[wi] = ow;
    }
}

// One launch for every width class (no serialisation of the u8 and u16 runs
// behind each other): blocks [0, nb1) decode the 8-bit runs, the next nb2
// blocks the 16-bit runs, the rest the 32-bit runs.  One warp per CTA, so
// the warps land on separate SMs.
template <int NB>
__device__ __forceinline__ void decode_runs(const RunDesc* __restrict__ runs, const uint32_t* __restrict__ rc_runs,
                                            int n, int blk, const PlaneRef* __restrict__ planes, uint32_t P) {
    const int lane = threadIdx.x;
    for (int b = 0; b < NB; b++)  // new_bittree_probs (_rc.py:304-317)
        for (uint32_t i = 0; i < 256; i++)
            sts_u32(node_addr(P + b * kTreeBytes, i), (i != 0 && (i & (i - 1)) == 0) ? 3686u : 2048u);
    const int gi = blk * kRPW + lane;
    if (gi >= n) return;
    const RunDesc r = runs[rc_runs[gi]];
    const uint32_t hw = (uint32_t)r.w * r.h;
    for (int f = 0; f < r.count; f++) {
        const PlaneRef pr = planes[r.plane_base + f];
        if (pr.mode != 0) continue;  // RAW plane (already copied to aligned storage)
        uint32_t* out = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(pr.samples));
        if (f > 0) {
            const uint32_t* prev = reinterpret_cast<const uint32_t*>(planes[r.plane_base + f - 1].samples);
            decode_plane<NB, true>(P, pr, prev, out, hw, r.w);
        } else {
            decode_plane<NB, false>(P, pr, nullptr, out, hw, r.w);
        }
    }
}

struct RcClasses {
    int n[3];    // runs per class (1, 2, 4 bytes per sample)
    int off[3];  // first index into rc_runs
    int blk[4];  // block prefix
};

__global__ void __launch_bounds__(kRPW) rc_decode_kernel(const RunDesc* __restrict__ runs,
                                                         const uint32_t* __restrict__ rc_runs, RcClasses c,
                                                         const PlaneRef* __restrict__ planes) {
    extern __shared__ uint4 probs_s[];
    const int b = blockIdx.x;
    const int nb = b < c.blk[1] ? 1 : (b < c.blk[2] ? 2 : 4);
    const uint32_t P = (uint32_t)__cvta_generic_to_shared(probs_s) + threadIdx.x * lane_stride(nb);
    if (b < c.blk[1]) decode_runs<1>(runs, rc_runs + c.off[0], c.n[0], b, planes, P);
    else if (b < c.blk[2]) decode_runs<2>(runs, rc_runs + c.off[1], c.n[1], b - c.blk[1], planes, P);
    else decode_runs<4>(runs, rc_runs + c.off[2], c.n[2], b - c.blk[2], planes, P);
}

void launch_rc_decode(const RunDesc* runs, const uint32_t* rc_runs, const int* n_per_class,
                      const PlaneRef* planes, cudaStream_t s) {
    RcClasses c;
    int nbmax = 0, off = 0;
    c.blk[0] = 0;
    for (int k = 0; k < 3; k++) {
        c.n[k] = n_per_class[k];
        c.off[k] = off;
        off += c.n[k];
        c.blk[k + 1] = c.blk[k] + (c.n[k] + kRPW - 1) / kRPW;
        if (c.n[k] > 0) nbmax = 1 << k;
    }
    if (c.blk[3] == 0) return;
    const size_t smem = (size_t)lane_stride(nbmax) * kRPW;
    cudaFuncSetAttribute(rc_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rc_decode_kernel<<<c.blk[3], kRPW, smem, s>>>(runs, rc_runs, c, planes);
}

}  // namespace gsv
