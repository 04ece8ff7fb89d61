// Per-frame render pipeline: project -> depth rank sort -> tile key emission
// -> tile sort -> tile ranges -> composite.  Everything is enqueued on one
// stream with counts kept on the device, so a frame needs no host round trip
// (the host only reads the counters back when asked for statistics or to
// detect a key-buffer overflow).
//
// Ordering contract (render.py:342-356): splats are composited in the order
// of np.argsort(depth, kind="stable") over project_set's survivors.  The
// depth sort below is a stable LSD radix sort of the fp64 depth bit patterns
// (depth > near > 0, so unsigned order == numeric order) with the splat index
// as payload over *all* splats in index order, culled splats keyed past the
// largest survivor: its first n_visible entries are exactly that order.  Tile
// keys are then emitted in rank order and stably sorted by tile, so every
// tile sees its splats in global depth-rank order.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>

#include "gsv_internal.h"
#include "sort.cuh"

namespace gsv {

void launch_project_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, cudaStream_t s,
                           int32_t* dbg_rect = nullptr, double* dbg_depth = nullptr);
void launch_splat2d(const Splat2DSrc& src, const CamDev& cam, RenderWork* w, cudaStream_t s);
void launch_project_soa(const SoaSrc& src, const CamDev& cam, RenderWork* w, int32_t* dbg_rect,
                        double* dbg_depth, cudaStream_t s);

enum { C_NVIS = 0, C_NKEYS = 1, C_DMIN = 2, C_DMAX = 3, C_OVF = 4, C_N = 5, C_KCLAMP = 6,
       C_RN = 7, C_NPASS = 8 /* int pair: passes, key shift */, C_MAXK = 9 /* sticky */,
       C_TOTK = 10, C_EMITK = 11, C_LONGRUNS = 12, C_TIETICKET = 13 };

CamDev make_cam(const gsv_camera& c) {
    CamDev d;
    memcpy(d.R, c.rotation, sizeof d.R);
    memcpy(d.t, c.translation, sizeof d.t);
    // center = -R^T @ t (render.py:74-77), evaluated like BLAS gemv
    for (int i = 0; i < 3; i++) {
        const double m0 = -c.rotation[0 * 3 + i], m1 = -c.rotation[1 * 3 + i], m2 = -c.rotation[2 * 3 + i];
        d.center[i] = fma(m2, c.translation[2], fma(m1, c.translation[1], m0 * c.translation[0]));
    }
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    d.near_ = c.near_plane;
    for (int k = 0; k < 3; k++) d.bg[k] = (float)c.background[k];
    d.width = c.width;
    d.height = c.height;
    return d;
}

// ---------------------------------------------------------------------------
// Per-frame reset: counters, the radix digit histograms the producers of the
// sort keys accumulate into (kHistRegions regions of 4 x 256), tile flags.
constexpr int kHistRegions = 4;  // depth sort, tile sort of round 1, 2 (+1 spare)
__global__ void __launch_bounds__(256) reset_frame_kernel(unsigned long long* ctr, long long n,
                                                          uint32_t* __restrict__ ghist,
                                                          uint32_t* __restrict__ tile_done, int ntiles,
                                                          uint32_t open_word) {
    for (int i = threadIdx.x; i < kHistRegions * 1024; i += 256) ghist[i] = 0;
    for (int i = threadIdx.x; i < ntiles; i += 256) tile_done[i] = open_word;
    if (threadIdx.x) return;
    ctr[C_NVIS] = 0;
    ctr[C_NKEYS] = 0;
    ctr[C_DMIN] = ~0ull;
    ctr[C_DMAX] = 0;
    ctr[C_OVF] = 0;
    ctr[C_N] = (unsigned long long)n;
    ctr[C_KCLAMP] = 0;
    ctr[C_RN] = 0;
    ctr[C_TOTK] = 0;
    ctr[C_EMITK] = 0;
    ctr[C_LONGRUNS] = 0;
    ctr[C_TIETICKET] = 0;
    reinterpret_cast<int*>(ctr + C_NPASS)[0] = 0;
    reinterpret_cast<int*>(ctr + C_NPASS)[1] = 0;
}

// Significant bits of the rebased depth key the radix sort runs on (24:
// three passes; ties of the truncated key are put in exact order by
// depth_tie_fixup).  GSV_DEPTH_KEY_BITS (16, 24 or 32) for dev tuning.
static int depth_key_bits() {
    static int b = 0;
    if (!b) {
        const char* e = getenv("GSV_DEPTH_KEY_BITS");
        b = e ? atoi(e) : 24;
        if (b != 16 && b != 24 && b != 32) b = 24;
    }
    return b;
}

// Rebase survivor depth bits to [0, range]; culled splats get range + 1 (so
// they sort last).  The radix sort runs on the top 32 significant bits of
// that key (key32); full[] keeps the 64-bit key by splat index for the
// fix-up of key32 ties.  Passes = bytes spanned by key32.
// Also accumulates the digit histograms of all 4 radix passes (fused
// radix_hist, sort.cuh).
__global__ void __launch_bounds__(256) depth_key_prep(uint64_t* __restrict__ full, uint32_t* __restrict__ key32,
                                                      unsigned long long* __restrict__ ctr,
                                                      uint32_t* __restrict__ ghist, int keybits) {
    __shared__ uint32_t h[4][256];
#pragma unroll
    for (int p = 0; p < 4; p++) h[p][threadIdx.x] = 0;
    __syncthreads();
    const uint64_t n = ctr[C_N];
    const uint64_t nvis = ctr[C_NVIS];
    const uint64_t lo = ctr[C_DMIN], hi = ctr[C_DMAX];
    const uint64_t dead = nvis ? (hi - lo) + 1 : 0;
    const int bits = dead ? 64 - __clzll((long long)dead) : 0;
    const int shift = bits > keybits ? bits - keybits : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int kb = bits - shift;
        reinterpret_cast<int*>(ctr + C_NPASS)[0] = (nvis == 0 || (nvis == n && hi == lo)) ? 0 : (kb + 7) / 8;
        reinterpret_cast<int*>(ctr + C_NPASS)[1] = shift;
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = full[i];
        const uint64_t r = (k == ~0ull) ? dead : k - lo;
        full[i] = r;
        const uint32_t k32 = (uint32_t)(r >> shift);
        key32[i] = k32;
#pragma unroll
        for (int p = 0; p < 4; p++) atomicAdd(&h[p][(k32 >> (8 * p)) & 0xFFu], 1u);
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; p++)
        if (h[p][threadIdx.x]) atomicAdd(&ghist[p * 256 + threadIdx.x], h[p][threadIdx.x]);
}

// Stable order among equal key32 values by the full key.  The radix sort is
// stable over splats in index order, so a run of equal key32 is in index
// order and its exact order is (full key, index).  A thread per run start
// finds the run's end by galloping (key32 is sorted); runs of up to 32 are
// put in order by that thread (insertion sort), longer runs -- many distinct
// depths sharing one truncated key, e.g. a far outlier stretching the depth
// range -- are listed for depth_tie_long (a CTA per run).
constexpr uint32_t kShortTieRun = 32;
__device__ void tie_sort_long_runs(uint32_t* __restrict__ idx, const uint64_t* __restrict__ full, uint32_t nruns,
                                   const uint32_t* __restrict__ long_runs, uint64_t* __restrict__ sk0,
                                   uint32_t* __restrict__ si0, uint64_t* __restrict__ sk1,
                                   uint32_t* __restrict__ si1);

__global__ void __launch_bounds__(256) depth_tie_fixup(const uint32_t* __restrict__ k0,
                                                       const uint32_t* __restrict__ k1, uint32_t* __restrict__ i0,
                                                       uint32_t* __restrict__ i1, const uint64_t* __restrict__ full,
                                                       unsigned long long* __restrict__ ctr,
                                                       uint32_t* __restrict__ long_runs, uint64_t* __restrict__ sk0,
                                                       uint32_t* __restrict__ si0, uint64_t* __restrict__ sk1,
                                                       uint32_t* __restrict__ si1) {
    const int np = reinterpret_cast<const int*>(ctr + C_NPASS)[0];
    const int shift = reinterpret_cast<const int*>(ctr + C_NPASS)[1];
    if (shift == 0 || np == 0) return;
    const uint32_t n = (uint32_t)ctr[C_N];
    const uint32_t* key = (np & 1) ? k1 : k0;
    uint32_t* idx = (np & 1) ? i1 : i0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const uint32_t k = key[r];
        if (r > 0 && key[r - 1] == k) continue;
        if (r + 1 >= n || key[r + 1] != k) continue;
        // upper bound of k in [r + 1, n): gallop, then bisect
        uint32_t lo = r + 1, step = 1, hi = r + 2;
        while (hi < n && key[hi] == k) {
            lo = hi;
            step *= 2;
            hi = (n - lo > step) ? lo + step : n;
        }
        while (hi - lo > 1) {  // key[lo] == k, key[hi] != k (or hi == n)
            const uint32_t m = lo + (hi - lo) / 2;
            if (key[m] == k) lo = m;
            else hi = m;
        }
        const uint32_t e = lo + 1;
        if (e - r > kShortTieRun) {
            const unsigned long long j = atomicAdd(ctr + C_LONGRUNS, 1ull);
            long_runs[2 * j] = r;
            long_runs[2 * j + 1] = e;
            continue;
        }
        const uint64_t f0 = full[idx[r]];
        bool same = true;
        for (uint32_t q = r + 1; q < e && same; q++) same = full[idx[q]] == f0;
        if (same) continue;
        for (uint32_t q = r + 1; q < e; q++) {
            const uint32_t v = idx[q];
            const uint64_t fv = full[v];
            uint32_t p = q;
            while (p > r && full[idx[p - 1]] > fv) {
                idx[p] = idx[p - 1];
                p--;
            }
            idx[p] = v;
        }
    }
    // the last CTA to finish sorts the listed long runs (rare: only when many
    // distinct depths share a truncated key); no extra launch per frame
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long t = atomicAdd(ctr + C_TIETICKET, 1ull);
        last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t nruns = (uint32_t)*reinterpret_cast<volatile unsigned long long*>(ctr + C_LONGRUNS);
    if (nruns) tie_sort_long_runs(idx, full, nruns, long_runs, sk0, si0, sk1, si1);
}

// (full key, index) order
__device__ __forceinline__ bool tie_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Long runs of equal key32: a CTA per run sorts (full key, index) pairs --
// bitonic in shared memory per chunk of kTieChunk, then merge passes between
// two global scratch buffers (merge path per thread) for longer runs.
constexpr int kTieThreads = 256, kTieChunk = 2048;
__device__ void tie_sort_long_runs(uint32_t* __restrict__ idx, const uint64_t* __restrict__ full, uint32_t nruns,
                                   const uint32_t* __restrict__ long_runs, uint64_t* __restrict__ sk0,
                                   uint32_t* __restrict__ si0, uint64_t* __restrict__ sk1,
                                   uint32_t* __restrict__ si1) {
    __shared__ uint64_t ks[kTieChunk];
    __shared__ uint32_t is[kTieChunk];
    for (uint32_t j = 0; j < nruns; j++) {
        const uint32_t r = long_runs[2 * j], e = long_runs[2 * j + 1], L = e - r;
        // 1) chunks of kTieChunk sorted in shared memory
        for (uint32_t c0 = 0; c0 < L; c0 += kTieChunk) {
            const uint32_t m = min((uint32_t)kTieChunk, L - c0);
            uint32_t P = 1;
            while (P < m) P *= 2;
            for (uint32_t t = threadIdx.x; t < P; t += kTieThreads) {
                if (t < m) {
                    const uint32_t v = idx[r + c0 + t];
                    is[t] = v;
                    ks[t] = full[v];
                } else {
                    is[t] = 0xFFFFFFFFu;
                    ks[t] = ~0ull;
                }
            }
            __syncthreads();
            for (uint32_t k = 2; k <= P; k *= 2)
                for (uint32_t h = k / 2; h > 0; h /= 2) {
                    for (uint32_t t = threadIdx.x; t < P / 2; t += kTieThreads) {
                        const uint32_t a = 2 * h * (t / h) + (t % h), b = a + h;
                        const bool up = (a & k) == 0;
                        const bool gt = tie_less(ks[b], is[b], ks[a], is[a]);
                        if (gt == up) {
                            const uint64_t tk = ks[a];
                            ks[a] = ks[b];
                            ks[b] = tk;
                            const uint32_t ti = is[a];
                            is[a] = is[b];
                            is[b] = ti;
                        }
                    }
                    __syncthreads();
                }
            for (uint32_t t = threadIdx.x; t < m; t += kTieThreads) {
                if (L <= (uint32_t)kTieChunk) {
                    idx[r + t] = is[t];
                } else {
                    sk0[r + c0 + t] = ks[t];
                    si0[r + c0 + t] = is[t];
                }
            }
            __syncthreads();
        }
        if (L <= (uint32_t)kTieChunk) continue;
        // 2) merge passes: runs of w -> 2w, ping-pong between the scratch pairs
        uint64_t* ka = sk0 + r;
        uint32_t* ia = si0 + r;
        uint64_t* kb = sk1 + r;
        uint32_t* ib = si1 + r;
        for (uint32_t w = kTieChunk; w < L; w *= 2) {
            for (uint32_t s0 = 0; s0 < L; s0 += 2 * w) {
                const uint32_t na = min(w, L - s0), nb = (L - s0 > w) ? min(w, L - s0 - w) : 0;
                const uint64_t* xk = ka + s0;
                const uint32_t* xi = ia + s0;
                const uint64_t* yk = xk + na;
                const uint32_t* yi = xi + na;
                const uint32_t tot = na + nb, per = (tot + kTieThreads - 1) / kTieThreads;
                const uint32_t o0 = min(tot, threadIdx.x * per), o1 = min(tot, o0 + per);
                if (o0 < o1) {
                    // merge path: first x index of the diagonal o0
                    uint32_t lo = o0 > nb ? o0 - nb : 0, hi = min(o0, na);
                    while (lo < hi) {
                        const uint32_t mi = (lo + hi) / 2;  // take x[mi] before y[o0 - 1 - mi]?
                        if (tie_less(yk[o0 - 1 - mi], yi[o0 - 1 - mi], xk[mi], xi[mi])) hi = mi;
                        else lo = mi + 1;
                    }
                    uint32_t x = lo, y = o0 - lo;
                    for (uint32_t o = o0; o < o1; o++) {
                        const bool tx = y >= nb || (x < na && tie_less(xk[x], xi[x], yk[y], yi[y]));
                        if (tx) {
                            kb[s0 + o] = xk[x];
                            ib[s0 + o] = xi[x];
                            x++;
                        } else {
                            kb[s0 + o] = yk[y];
                            ib[s0 + o] = yi[y];
                            y++;
                        }
                    }
                }
            }
            __syncthreads();
            uint64_t* tk = ka;
            ka = kb;
            kb = tk;
            uint32_t* ti = ia;
            ia = ib;
            ib = ti;
        }
        for (uint32_t t = threadIdx.x; t < L; t += kTieThreads) idx[r + t] = ia[t];
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t rec_tile_count(const SplatRec& r) {
    const uint32_t x0 = r.rx & 0xFFFFu, x1 = r.rx >> 16, y0 = r.ry & 0xFFFFu, y1 = r.ry >> 16;
    return ((x1 - 1) / kTile - x0 / kTile + 1) * ((y1 - 1) / kTile - y0 / kTile + 1);
}

// Round [a, b) of the depth ranks: count the not-yet-saturated tiles each
// splat overlaps, turn the counts into offsets with a single-pass
// decoupled-look-back scan across CTAs (ticketed CTA order, epoch-tagged
// status words so nothing needs resetting between uses), and scatter the
// (tile, rank) keys in rank order -- one launch instead of count + scan +
// emit.
constexpr int kEmitThreads = 256, kEmitPer = 1, kEmitTile = kEmitThreads * kEmitPer;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned long long st_pack(uint32_t epoch, uint32_t flag, unsigned long long v) {
    return ((unsigned long long)(epoch & 0xFFFFFFu) << 40) | ((unsigned long long)flag << 38) | v;
}

// Bit t of the open-tile mask is set while tile t has a strip not yet
// saturated (the emission of later rounds only visits those tiles).
__global__ void open_mask_kernel(const uint32_t* __restrict__ tile_done, int ntiles, uint32_t* __restrict__ mask) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const bool open = t < ntiles && tile_done[t] != kTileAllSat;
    const uint32_t b = __ballot_sync(0xffffffffu, open);
    if ((threadIdx.x & 31) == 0 && t < ntiles) mask[t >> 5] = b;
}

// number of set bits of mask in [lo, hi] (tile ids)
__device__ __forceinline__ uint32_t mask_count(const uint32_t* m, uint32_t lo, uint32_t hi) {
    uint32_t c = 0;
    for (uint32_t w = lo >> 5; w <= (hi >> 5); w++) {
        uint32_t v = m[w];
        if (w == (lo >> 5)) v &= 0xFFFFFFFFu << (lo & 31);
        if (w == (hi >> 5)) v &= 0xFFFFFFFFu >> (31 - (hi & 31));
        c += __popc(v);
    }
    return c;
}

constexpr int kMaskWordsSmem = 2048;  // open-tile masks of up to 65536 tiles live in shared memory

__global__ void __launch_bounds__(kEmitThreads) round_emit_fused(
    const uint2* __restrict__ rect, const uint32_t* __restrict__ didx0, const uint32_t* __restrict__ didx1,
    unsigned long long* __restrict__ ctr, uint32_t a, uint32_t b,
    const uint32_t* __restrict__ open_mask, int ntiles, uint32_t* __restrict__ tkey,
    uint32_t* __restrict__ tval, uint64_t cap, int ntx, unsigned long long* __restrict__ status,
    unsigned int* __restrict__ ticket, uint32_t epoch, uint32_t* __restrict__ ghist, int tpasses) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_hist[4][256];
    __shared__ uint32_t s_mask[kMaskWordsSmem];
    __shared__ unsigned long long s_prefix;
    __shared__ uint32_t s_wsum[kEmitThreads / 32];
    if (threadIdx.x == 0) {
        const uint32_t t = atomicAdd(ticket, 1u);
        if (t == gridDim.x - 1) *ticket = 0;  // every CTA has its ticket: reset for the next use
        s_tile = t;
    }
#pragma unroll
    for (int p = 0; p < 4; p++) s_hist[p][threadIdx.x] = 0;
    // all tiles open (first round): open_mask == nullptr
    const int nwords = (ntiles + 31) >> 5;
    const bool mask_in_smem = open_mask && nwords <= kMaskWordsSmem;
    if (mask_in_smem)
        for (int w = threadIdx.x; w < nwords; w += kEmitThreads) s_mask[w] = open_mask[w];
    const uint32_t* mask = mask_in_smem ? s_mask : open_mask;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t nvis = (uint32_t)ctr[C_NVIS];
    const uint32_t hi = b < nvis ? b : nvis;
    const uint32_t m = hi > a ? hi - a : 0;
    const uint32_t nt = (m + kEmitTile - 1) / kEmitTile;
    if (tile >= nt) {
        if (tile == 0 && threadIdx.x == 0) {  // empty round
            ctr[C_NKEYS] = 0;
            ctr[C_KCLAMP] = 0;
        }
        return;
    }
    static_assert(kEmitPer == 1, "one splat per thread");
    const uint32_t base = tile * kEmitTile + threadIdx.x;
    uint32_t x0 = 1, x1 = 0, y0 = 1, y1 = 0;  // this thread's splat, tile coordinates (inclusive)
    uint32_t sum = 0;
    // depth rank -> splat: the sort's index buffer (the pass count decides
    // which ping-pong half holds it); keys carry the splat index, so the
    // compositor reads the records where the projection wrote them
    const uint32_t* order = (reinterpret_cast<const int*>(ctr + C_NPASS)[0] & 1) ? didx1 : didx0;
    uint32_t sidx = 0;
    if (base < m) {
        sidx = __ldg(order + a + base);
        const uint2 r = __ldg(rect + sidx);
        x0 = (r.x & 0xFFFFu) / kTile;
        x1 = ((r.x >> 16) - 1) / kTile;
        y0 = (r.y & 0xFFFFu) / kTile;
        y1 = ((r.y >> 16) - 1) / kTile;
        if (!mask) {
            sum = (x1 - x0 + 1) * (y1 - y0 + 1);
        } else {
            for (uint32_t ty = y0; ty <= y1; ty++) sum += mask_count(mask, ty * ntx + x0, ty * ntx + x1);
        }
    }
    // block exclusive scan of the per-thread sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t wb = 0, total = 0;
    for (int w = 0; w < kEmitThreads / 32; w++) {
        if (w < warp) wb += s_wsum[w];
        total += s_wsum[w];
    }
    const uint32_t excl = wb + x - sum;
    if (warp == 0) {
        // decoupled look-back, 32 predecessors per step (one per lane)
        unsigned long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(status, st_pack(epoch, 2, total));
        } else {
            if (lane == 0) atomicExch(status + tile, st_pack(epoch, 1, total));
            const uint32_t ep = epoch & 0xFFFFFFu;
            int j = (int)tile - 1;
            for (;;) {
                const int idx = j - lane;
                const unsigned long long wv = idx >= 0 ? ld_volatile_u64(status + idx) : st_pack(epoch, 2, 0);
                const uint32_t fl = (uint32_t)(wv >> 38) & 3u;
                const bool valid = (uint32_t)(wv >> 40) == ep && fl != 0;
                const uint32_t inv = __ballot_sync(0xffffffffu, !valid);
                const uint32_t inc = __ballot_sync(0xffffffffu, valid && fl == 2);
                // lanes [0, k) are consumed this step
                const uint32_t first_inv = inv ? (uint32_t)(__ffs(inv) - 1) : 32u;
                const uint32_t first_inc = inc ? (uint32_t)(__ffs(inc) - 1) : 32u;
                const bool done = first_inc < first_inv;
                const uint32_t k = done ? first_inc + 1 : first_inv;
                unsigned long long v = (uint32_t)lane < k ? (wv & ((1ull << 38) - 1)) : 0ull;
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (done) break;
                j -= (int)k;
                if (k == 0) __nanosleep(32);
            }
            if (lane == 0) atomicExch(status + tile, st_pack(epoch, 2, prefix + total));
        }
        if (lane == 0) s_prefix = prefix;
        if (lane == 0 && tile == nt - 1) {
            const unsigned long long K = prefix + total;
            ctr[C_NKEYS] = K;
            ctr[C_KCLAMP] = K < cap ? K : cap;
            if (K > cap) ctr[C_OVF] = K;
            atomicMax(ctr + C_MAXK, K);
            ctr[C_EMITK] += K;
        }
    }
    __syncthreads();
    // scatter this thread's splat's keys in rank order (open tiles only)
    if (sum) {
        unsigned long long o = s_prefix + excl;
        const uint32_t r = sidx;
        for (uint32_t ty = y0; ty <= y1; ty++)
            for (uint32_t tx = x0; tx <= x1; tx++) {
                const uint32_t t = ty * (uint32_t)ntx + tx;
                if (mask && !((mask[t >> 5] >> (t & 31)) & 1u)) continue;
                if (o < cap) {
                    tkey[o] = t;
                    tval[o] = r;
                    for (int p = 0; p < tpasses; p++) atomicAdd(&s_hist[p][(t >> (8 * p)) & 0xFFu], 1u);
                }
                o++;
            }
    }
    __syncthreads();
    for (int p = 0; p < tpasses; p++)
        if (s_hist[p][threadIdx.x]) atomicAdd(&ghist[p * 256 + threadIdx.x], s_hist[p][threadIdx.x]);
}

// sorted tile keys -> tile range offsets off[t] = first key index >= t
// (t = 0..ntiles): key i fills the tiles in (key[i-1], key[i]]
__global__ void keys_to_off_kernel(const uint32_t* __restrict__ key, const unsigned long long* __restrict__ ctr,
                                   int ntiles, uint32_t* __restrict__ off) {
    const uint32_t K = (uint32_t)ctr[C_KCLAMP];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= K; i += gridDim.x * blockDim.x) {
        const uint32_t lo = i == 0 ? 0u : __ldg(key + i - 1) + 1u;
        const uint32_t hi = i == K ? (uint32_t)ntiles : __ldg(key + i);
        for (uint32_t t = lo; t <= hi; t++) off[t] = i;
    }
}

// ---------------------------------------------------------------------------
// First round without a sort.  Every tile is open in round 1, so the
// (tile, splat) pairs of ranks [a, b) are binned directly, in rank order
// inside each tile, by counting: the ranks are cut into blocks of B; (1) per
// block, the tiles each splat's rect covers are counted in shared memory;
// (2) per tile, the block counts are turned into exclusive offsets and the
// tile totals into the tile ranges; (3) per block, ONE warp walks its splats
// in rank order and places each splat index at its tiles' next slot.  The
// compositor then reads each tile's range directly (no tile keys, no search).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rect_tiles_of(const uint2* __restrict__ rect, uint32_t idx, uint32_t& tx0,
                                              uint32_t& tx1, uint32_t& ty0, uint32_t& ty1) {
    const uint2 rr = __ldg(rect + idx);
    const uint32_t rx = rr.x, ry = rr.y;
    tx0 = (rx & 0xFFFFu) / kTile;
    tx1 = ((rx >> 16) - 1) / kTile;
    ty0 = (ry & 0xFFFFu) / kTile;
    ty1 = ((ry >> 16) - 1) / kTile;
}

__global__ void __launch_bounds__(256) r1_count_kernel(const uint2* __restrict__ rect,
                                                       const uint32_t* __restrict__ didx0,
                                                       const uint32_t* __restrict__ didx1,
                                                       const unsigned long long* __restrict__ ctr, uint32_t a,
                                                       uint32_t b, uint32_t B, int ntx, int ntiles,
                                                       const uint32_t* __restrict__ mask, uint32_t* __restrict__ bc) {
    extern __shared__ uint32_t s_cnt[];
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_cnt[t] = 0;
    __syncthreads();
    const uint32_t nvis = (uint32_t)ctr[C_NVIS];
    const uint32_t hi = min(b, nvis);
    const uint32_t* order = (reinterpret_cast<const int*>(ctr + C_NPASS)[0] & 1) ? didx1 : didx0;
    const uint32_t r0 = a + blockIdx.x * B, r1 = min(r0 + B, hi);
    for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        uint32_t tx0, tx1, ty0, ty1;
        rect_tiles_of(rect, __ldg(order + r), tx0, tx1, ty0, ty1);
        for (uint32_t ty = ty0; ty <= ty1; ty++)
            for (uint32_t tx = tx0; tx <= tx1; tx++) {
                const uint32_t t = ty * (uint32_t)ntx + tx;
                if (!mask || ((__ldg(mask + (t >> 5)) >> (t & 31)) & 1u)) atomicAdd(&s_cnt[t], 1u);
            }
    }
    __syncthreads();
    uint32_t* row = bc + (size_t)blockIdx.x * ntiles;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) row[t] = s_cnt[t];
}

// per tile: block counts -> exclusive offsets inside the tile (in place),
// tile totals -> off[t].  A CTA takes 32 tiles (one per lane: coalesced
// 128-B rows) and all blocks, 32 consecutive blocks per warp; the loads of
// a warp's 32 blocks are independent (all in flight at once)
__global__ void __launch_bounds__(512) r1_scan_blocks_kernel(uint32_t* __restrict__ bc, int nblk, int ntiles,
                                                             uint32_t* __restrict__ off) {
    __shared__ uint32_t s_tot[16][32];
    const int nw = blockDim.x >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int k0 = warp * 32;
    uint32_t v[32];
#pragma unroll
    for (int k = 0; k < 32; k++) v[k] = (t < ntiles && k0 + k < nblk) ? bc[(size_t)(k0 + k) * ntiles + t] : 0u;
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) {
        const uint32_t x = v[k];
        v[k] = run;
        run += x;
    }
    s_tot[warp][lane] = run;
    __syncthreads();
    uint32_t base = 0, tot = 0;
    for (int w = 0; w < nw; w++) {
        base += w < warp ? s_tot[w][lane] : 0u;
        tot += s_tot[w][lane];
    }
    if (t < ntiles) {
#pragma unroll
        for (int k = 0; k < 32; k++)
            if (k0 + k < nblk) bc[(size_t)(k0 + k) * ntiles + t] = base + v[k];
        if (warp == 0) off[t] = tot;
    }
}

// exclusive scan of the tile totals (one CTA), key counters as the emission
// would set them (capacity check and re-render on overflow)
__global__ void __launch_bounds__(1024) r1_scan_tiles_kernel(uint32_t* __restrict__ off, int ntiles,
                                                             unsigned long long* __restrict__ ctr, uint64_t cap) {
    __shared__ uint32_t s_w[32];
    // up to 32 tiles per thread (32768 tiles: 4K is 32400), loaded at once
    constexpr int kPer = 32;
    const int per = (ntiles + 1023) / 1024;
    const int t0 = threadIdx.x * per;
    uint32_t v[kPer];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; i++) {
        v[i] = (i < per && t0 + i < ntiles) ? off[t0 + i] : 0u;
        sum += v[i];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = s_w[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        s_w[lane] = v;
    }
    __syncthreads();
    uint32_t run = (warp ? s_w[warp - 1] : 0u) + x - sum;
#pragma unroll
    for (int i = 0; i < kPer; i++)
        if (i < per && t0 + i < ntiles) {
            off[t0 + i] = run;
            run += v[i];
        }
    if (threadIdx.x == 1023) {
        const unsigned long long K = s_w[31];
        off[ntiles] = (uint32_t)K;
        ctr[C_NKEYS] = K;
        ctr[C_KCLAMP] = K < cap ? K : cap;
        if (K > cap) ctr[C_OVF] = K;
        atomicMax(ctr + C_MAXK, K);
        ctr[C_EMITK] += K;
    }
}

// one warp per block of ranks: splats in rank order, each one's tiles
// spread over the lanes; a tile's next slot lives in shared memory
// LANEPAR (default): the warp places 32 consecutive splats at once, a lane
// per splat.  Per batch each lane ORs its bit into per-column and per-row
// lane masks of the rect it covers (shared memory); a (splat, tile) pair's
// slot is then the tile's next slot plus the number of lower lanes covering
// the tile -- popc(colmask[tx] & rowmask[ty] & lanes below) -- so the
// order within a tile is still rank order, and the lowest covering lane
// advances the tile's next slot by the batch's count.  No splat waits for
// the one before it (the sequential walk chains ~200 cycles per splat).
template <bool LANEPAR>
__global__ void __launch_bounds__(256) r1_place_kernel(const uint2* __restrict__ rect,
                                                      const uint32_t* __restrict__ didx0,
                                                      const uint32_t* __restrict__ didx1,
                                                      const unsigned long long* __restrict__ ctr, uint32_t a,
                                                      uint32_t b, uint32_t B, int ntx, int ntiles,
                                                      const uint32_t* __restrict__ bc,
                                                      const uint32_t* __restrict__ off, uint32_t* __restrict__ val,
                                                      uint64_t cap, const uint32_t* __restrict__ mask) {
    extern __shared__ uint32_t s_next[];
    const uint32_t* row = bc + (size_t)blockIdx.x * ntiles;
    for (int t0 = threadIdx.x; t0 < ntiles; t0 += 4 * blockDim.x) {  // 4 independent pairs in flight
        uint32_t o4[4], r4[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int t = t0 + u * blockDim.x;
            o4[u] = t < ntiles ? __ldg(off + t) : 0u;
            r4[u] = t < ntiles ? __ldg(row + t) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (t0 + u * (int)blockDim.x < ntiles) s_next[t0 + u * blockDim.x] = o4[u] + r4[u];
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;  // the placement itself is one warp, in rank order
    const uint32_t nvis = (uint32_t)ctr[C_NVIS];
    const uint32_t hi = min(b, nvis);
    const uint32_t* order = (reinterpret_cast<const int*>(ctr + C_NPASS)[0] & 1) ? didx1 : didx0;
    const uint32_t r0 = a + blockIdx.x * B, r1 = min(r0 + B, hi);
    const int lane = threadIdx.x;
    // 32 splats' rects at a time (the next 32 loaded while these are
    // placed), then one splat after the other
    uint32_t nidx = 0, nrx = 0, nry = 0;
    auto fetch = [&](uint32_t base) {
        const uint32_t rr = base + lane;
        nidx = 0;
        nrx = nry = 0;
        if (rr < r1) {
            nidx = __ldg(order + rr);
            const uint2 q = __ldg(rect + nidx);
            nrx = q.x;
            nry = q.y;
        }
    };
    if (r0 < r1) fetch(r0);
    if constexpr (LANEPAR) {
        __shared__ uint32_t s_colm[256], s_rowm[256];  // lane masks per tile column / row
        for (int k = lane; k < 256; k += 32) s_colm[k] = s_rowm[k] = 0u;
        __syncwarp();
        const uint32_t below = (1u << lane) - 1u;
        for (uint32_t base = r0; base < r1; base += 32) {
            const uint32_t idx = nidx, rx = nrx, ry = nry;
            if (base + 32 < r1) fetch(base + 32);
            bool act = base + lane < r1;
            const uint32_t tx0 = (rx & 0xFFFFu) / kTile, tx1 = ((rx >> 16) - 1) / kTile;
            const uint32_t ty0 = (ry & 0xFFFFu) / kTile, ty1 = ((ry >> 16) - 1) / kTile;
            if (act && mask) {  // later rounds: splats whose tiles are all closed place nothing
                uint32_t open = 0;
                for (uint32_t ty = ty0; ty <= ty1 && !open; ty++) open = mask_count(mask, ty * ntx + tx0, ty * ntx + tx1);
                act = open != 0;
            }
            if (act) {
                for (uint32_t tx = tx0; tx <= tx1; tx++) atomicOr(&s_colm[tx], 1u << lane);
                for (uint32_t ty = ty0; ty <= ty1; ty++) atomicOr(&s_rowm[ty], 1u << lane);
            }
            __syncwarp();
            if (act) {  // slots: the tile's next slot + the lower lanes covering it
                for (uint32_t ty = ty0; ty <= ty1; ty++) {
                    const uint32_t rm = s_rowm[ty];
                    for (uint32_t tx = tx0; tx <= tx1; tx++) {
                        const uint32_t t = ty * (uint32_t)ntx + tx;
                        if (mask && !((__ldg(mask + (t >> 5)) >> (t & 31)) & 1u)) continue;
                        const uint32_t pos = s_next[t] + __popc(s_colm[tx] & rm & below);
                        if (pos < cap) val[pos] = idx;
                    }
                }
            }
            __syncwarp();
            if (act) {  // the lowest covering lane advances the tile by the batch's count
                for (uint32_t ty = ty0; ty <= ty1; ty++) {
                    const uint32_t rm = s_rowm[ty];
                    for (uint32_t tx = tx0; tx <= tx1; tx++) {
                        const uint32_t cov = s_colm[tx] & rm;
                        if ((cov & below) == 0u) s_next[ty * (uint32_t)ntx + tx] += __popc(cov);
                    }
                }
            }
            __syncwarp();
            if (act) {
                for (uint32_t tx = tx0; tx <= tx1; tx++) s_colm[tx] = 0u;
                for (uint32_t ty = ty0; ty <= ty1; ty++) s_rowm[ty] = 0u;
            }
            __syncwarp();
        }
        return;
    }
    for (uint32_t base = r0; base < r1; base += 32) {
        const uint32_t idx = nidx, rx = nrx, ry = nry;
        if (base + 32 < r1) fetch(base + 32);
        // per lane, for its own splat (off the sequential chain): first tile,
        // rect width and area in tiles, and the multiplier of k / w
        uint32_t t0 = 0, w = 1, area = 0, mw = 0;
        if (base + lane < r1) {
            const uint32_t tx0 = (rx & 0xFFFFu) / kTile, tx1 = ((rx >> 16) - 1) / kTile;
            const uint32_t ty0 = (ry & 0xFFFFu) / kTile, ty1 = ((ry >> 16) - 1) / kTile;
            t0 = ty0 * (uint32_t)ntx + tx0;
            w = tx1 - tx0 + 1;
            area = w * (ty1 - ty0 + 1);
            // k / w as one multiply-high, exact for k * w < 2^32 (w = 1:
            // the multiplier would be 2^32, handled apart)
            mw = w > 1 ? 0xFFFFFFFFu / w + 1u : 0u;
            if (mask) {  // later rounds: splats whose tiles are all closed place nothing
                uint32_t open = 0;
                for (uint32_t ty = ty0; ty <= ty1 && !open; ty++)
                    open = mask_count(mask, ty * ntx + tx0, ty * ntx + tx1);
                if (!open) area = 0;
            }
        }
        for (uint32_t todo = __ballot_sync(0xffffffffu, area != 0); todo; todo &= todo - 1) {
            const int q = __ffs(todo) - 1;
            const uint32_t sidx = __shfl_sync(0xffffffffu, idx, q), qt0 = __shfl_sync(0xffffffffu, t0, q);
            const uint32_t qw = __shfl_sync(0xffffffffu, w, q), qa = __shfl_sync(0xffffffffu, area, q);
            const uint32_t qm = __shfl_sync(0xffffffffu, mw, q);
            for (uint32_t k = lane; k < qa; k += 32) {
                const uint32_t dy = qw > 1 ? __umulhi(k, qm) : k, dx = k - dy * qw;
                const uint32_t t = qt0 + dy * (uint32_t)ntx + dx;
                if (mask && !((__ldg(mask + (t >> 5)) >> (t & 31)) & 1u)) continue;
                const uint32_t pos = s_next[t]++;
                if (pos < cap) val[pos] = sidx;
            }
            __syncwarp();
        }
    }
}


// ---------------------------------------------------------------------------
static void free_ptr(void* p) {
    if (p) cudaFree(p);
}

void work_free(RenderWork* w) {
    for (int b = 0; b < 2; b++) {
        free_ptr(w->dkey[b]);
        free_ptr(w->didx[b]);
        free_ptr(w->tkey[b]);
        free_ptr(w->tval[b]);
    }
    free_ptr(w->rec);
    free_ptr(w->rect);
    free_ptr(w->tie_k);
    free_ptr(w->tie_runs);
    free_ptr(w->state);
    free_ptr(w->tile_done);
    free_ptr(w->open_mask);
    free_ptr(w->r1_bc);
    free_ptr(w->r1_off);
    free_ptr(w->status);
    free_ptr(w->sort_ghist);
    free_ptr(w->sort_status);
    free_ptr(w->ctr);
    if (w->h_ctr) cudaFreeHost(w->h_ctr);
    *w = RenderWork();
}

int work_reserve(RenderWork* w, int64_t n, int64_t k, int tiles, int64_t npix) {
    if (!w->ctr) {
        GSV_CUDA(cudaMalloc(&w->ctr, kCtrWords * sizeof(unsigned long long)));
        GSV_CUDA(cudaMallocHost(&w->h_ctr, kCtrWords * sizeof(unsigned long long)));
        GSV_CUDA(cudaMemset(w->ctr, 0, kCtrWords * sizeof(unsigned long long)));
        memset(w->h_ctr, 0, kCtrWords * sizeof(unsigned long long));
    }
    n = std::max<int64_t>(n, 1);
    if (n > w->cap_n) {
        const int64_t c = std::max<int64_t>(n, w->cap_n * 5 / 4);
        for (int b = 0; b < 2; b++) {
            free_ptr(w->dkey[b]);
            free_ptr(w->didx[b]);
            GSV_CUDA(cudaMalloc(&w->dkey[b], c * sizeof(uint64_t)));
            GSV_CUDA(cudaMalloc(&w->didx[b], c * sizeof(uint32_t)));
        }
        free_ptr(w->rec);
        GSV_CUDA(cudaMalloc(&w->rec, c * sizeof(SplatRec)));
        free_ptr(w->rect);
        GSV_CUDA(cudaMalloc(&w->rect, c * sizeof(uint2)));
        free_ptr(w->tie_k);
        free_ptr(w->tie_runs);
        GSV_CUDA(cudaMalloc(&w->tie_k, c * sizeof(uint64_t)));
        GSV_CUDA(cudaMalloc(&w->tie_runs, (c / (kShortTieRun + 1) + 1) * 2 * sizeof(uint32_t)));
        free_ptr(w->status);
        const size_t ns = (size_t)(c / 256 + 4) * sizeof(unsigned long long) + 64;
        GSV_CUDA(cudaMalloc(&w->status, ns));
        GSV_CUDA(cudaMemset(w->status, 0, ns));
        w->ticket = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(w->status) + ns - 64);
        w->cap_n = c;
    }
    k = std::max<int64_t>(k, 1 << 16);
    if (k > w->cap_k) {
        const int64_t c = std::max<int64_t>(k, w->cap_k * 5 / 4);
        for (int b = 0; b < 2; b++) {
            free_ptr(w->tkey[b]);
            free_ptr(w->tval[b]);
            GSV_CUDA(cudaMalloc(&w->tkey[b], c * sizeof(uint32_t)));
            GSV_CUDA(cudaMalloc(&w->tval[b], c * sizeof(uint32_t)));
        }
        w->cap_k = c;
    }
    if (tiles > w->cap_tiles) {
        free_ptr(w->tile_done);
        free_ptr(w->open_mask);
        GSV_CUDA(cudaMalloc(&w->tile_done, (size_t)tiles * 4));
        GSV_CUDA(cudaMalloc(&w->open_mask, ((size_t)tiles + 31) / 32 * 4 + 4));
        w->cap_tiles = tiles;
    }
    if (npix > w->cap_pix) {
        free_ptr(w->state);
        GSV_CUDA(cudaMalloc(&w->state, (size_t)npix * sizeof(float4)));
        w->cap_pix = npix;
    }
    if (!w->sort_ghist) {
        GSV_CUDA(cudaMalloc(&w->sort_ghist, (kHistRegions * 1024 + 32) * sizeof(uint32_t)));
        GSV_CUDA(cudaMemset(w->sort_ghist, 0, (kHistRegions * 1024 + 32) * sizeof(uint32_t)));
    }
    const int64_t sw = radix_status_words(std::max(w->cap_n, w->cap_k));
    if (sw > w->sort_status_cap) {
        free_ptr(w->sort_status);
        GSV_CUDA(cudaMalloc(&w->sort_status, sw * sizeof(unsigned long long)));
        GSV_CUDA(cudaMemset(w->sort_status, 0, sw * sizeof(unsigned long long)));
        w->sort_status_cap = sw;
    }
    return GSV_OK;
}

static SortScratch sort_scratch(RenderWork* w) {
    return SortScratch{w->sort_ghist, w->sort_status,
                       reinterpret_cast<unsigned int*>(w->sort_ghist + kHistRegions * 1024), &w->sort_epoch};
}

// the tile_done word of a fresh tile: its strips open, the unused bytes saturated
static uint32_t open_word(int rows) {
    const int strips = 16 / (2 * rows);
    uint32_t w = 0;
    for (int k = strips; k < 4; k++) w |= (uint32_t)kTileSaturated << (8 * k);
    return w;
}

static unsigned prep_grid(int64_t n) { return (unsigned)std::min<int64_t>((n + 1023) / 1024, 148 * 2); }

// round-1 counting placement (dev toggle GSV_R1_BIN=0: emit + tile sort as in later rounds)
static bool r1_binning() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GSV_R1_BIN");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

// later rounds binned the same way, open tiles only (dev toggle GSV_R2_BIN=1;
// measured 7% slower than emit + sort: round 2's ~270k splats mostly place
// nothing, and the sequential warp still walks them)
static bool later_binning() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GSV_R2_BIN");
        v = e ? atoi(e) : 0;
    }
    return v != 0;
}

static uint32_t r1_block() {  // dev knob GSV_R1_BLOCK: minimum ranks per block (64, 32 measured 7% slower)
    static int v = 0;
    if (!v) {
        const char* e = getenv("GSV_R1_BLOCK");
        v = e ? atoi(e) : 128;
        if (v < 32) v = 32;
    }
    return (uint32_t)v;
}

static bool later_ranges() {  // dev toggle GSV_R2_RANGES
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GSV_R2_RANGES");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

// Dynamic shared memory above 48 KB for the round-1 binning kernels.  The
// attribute is per device, so the largest size unlocked so far is tracked per
// device (atomically: several host threads may render on one device).
// round-1 placement variant: GSV_R1_PLACE=2 the lane-parallel batches
// (frames up to 256 tile columns and rows), else the sequential walk
// (default: the lane-parallel form is bit-identical but measured ~1% slower
// in the frame-parallel steady state -- the lanes' rects differ in size, so
// a batch runs as long as its largest rect, twice)
static int r1_place_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GSV_R1_PLACE");
        v = e ? atoi(e) : 1;
    }
    return v;
}

static void launch_r1_place(uint32_t nblk, size_t sm, cudaStream_t s, const uint2* rect, const uint32_t* d0,
                            const uint32_t* d1, const unsigned long long* ctr, uint32_t a, uint32_t b, uint32_t B,
                            int ntx, int ntiles, const uint32_t* bc, const uint32_t* off, uint32_t* val,
                            uint64_t cap, const uint32_t* mask) {
    const int nty = ntiles / ntx;
    if (r1_place_variant() != 1 && ntx <= 256 && nty <= 256)
        r1_place_kernel<true><<<nblk, 256, sm, s>>>(rect, d0, d1, ctr, a, b, B, ntx, ntiles, bc, off, val, cap, mask);
    else
        r1_place_kernel<false><<<nblk, 256, sm, s>>>(rect, d0, d1, ctr, a, b, B, ntx, ntiles, bc, off, val, cap, mask);
}

static int r1_smem_attr(size_t sm) {
    if (sm + 2048 <= 48 * 1024) return GSV_OK;  // + the lane-parallel placement's 2 KB of static masks
    static std::atomic<size_t> unlocked[kMaxDevices];
    int dev = 0;
    GSV_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) return fail(GSV_E_CUDA, "device ordinal out of range");
    size_t cur = unlocked[dev].load();
    if (sm <= cur) return GSV_OK;
    GSV_CUDA(cudaFuncSetAttribute(r1_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    GSV_CUDA(cudaFuncSetAttribute(r1_place_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    GSV_CUDA(cudaFuncSetAttribute(r1_place_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    while (cur < sm && !unlocked[dev].compare_exchange_weak(cur, sm)) {
    }
    return GSV_OK;
}

static int r1_reserve(RenderWork* w, size_t bc_words, size_t off_words) {
    if (bc_words > w->r1_bc_cap) {
        free_ptr(w->r1_bc);
        w->r1_bc = nullptr;
        const size_t c = std::max(bc_words, w->r1_bc_cap * 5 / 4);
        GSV_CUDA(cudaMalloc(&w->r1_bc, c * 4));
        w->r1_bc_cap = c;
    }
    if (off_words > w->r1_off_cap) {
        free_ptr(w->r1_off);
        w->r1_off = nullptr;
        GSV_CUDA(cudaMalloc(&w->r1_off, off_words * 4));
        w->r1_off_cap = off_words;
    }
    return GSV_OK;
}

static int tile_passes(int ntiles) {
    int bits = 0;
    while ((1 << bits) < ntiles) bits++;
    return std::max(1, (bits + 7) / 8);
}

// Depth-rank rounds: [0, R1) for every tile, then [R1, n) only for the tiles
// still open.  Tiles saturate within the first ~10-30k ranks at config 2
// (~97 evaluations per covered pixel), so the second round
// emits keys only for the few tiles that never saturate: 1.08M keys instead
// of 7.18M at config 2 (measured with the oracle, tools/analysis notes in
// DESIGN.md).
static void round_bounds(int64_t n, std::vector<uint32_t>* b) {
    b->clear();
    b->push_back(0);
    static std::vector<int64_t> fixed;  // dev tuning: GSV_ROUNDS="r1,r2,..." (absolute ranks)
    static int init = 0;
    if (!init) {
        if (const char* e = getenv("GSV_ROUNDS")) {
            for (const char* q = e; *q;) {
                fixed.push_back(atoll(q));
                while (*q && *q != ',') q++;
                if (*q == ',') q++;
            }
        }
        init = 1;
    }
    if (!fixed.empty()) {
        for (int64_t r : fixed)
            if (r > (int64_t)b->back() && r < n) b->push_back((uint32_t)r);
    } else {
        const int64_t r1 = std::max<int64_t>(32768, n / 10);
        if (n > r1) b->push_back((uint32_t)r1);
    }
    b->push_back((uint32_t)std::max<int64_t>(n, 0));
}

// Dev diagnostics: GSV_DEBUG_SKIP lists stages whose kernels are not
// launched (composite, tsort, dsort, emit) -- wrong images, used only to
// measure what each stage costs in the frame-parallel steady state.
static unsigned debug_double() {  // GSV_DEBUG_DOUBLE: stages launched twice (marginal cost probe)
    static int init = 0;
    static unsigned mask = 0;
    if (!init) {
        if (const char* e = getenv("GSV_DEBUG_DOUBLE")) {
            if (strstr(e, "composite")) mask |= 1;
            if (strstr(e, "tsort")) mask |= 2;
            if (strstr(e, "dsort")) mask |= 4;
            if (strstr(e, "emit")) mask |= 8;
            if (strstr(e, "project")) mask |= 16;
            if (strstr(e, "gather")) mask |= 32;
            if (strstr(e, "fixup")) mask |= 64;
            if (strstr(e, "lastround")) mask |= 128;
            if (strstr(e, "r1count")) mask |= 256;
            if (strstr(e, "r1place")) mask |= 512;
        }
        init = 1;
    }
    return mask;
}

static unsigned debug_skip() {
    static int init = 0;
    static unsigned mask = 0;
    if (!init) {
        const char* e = getenv("GSV_DEBUG_SKIP");
        if (e) {
            if (strstr(e, "composite")) mask |= 1;
            if (strstr(e, "tsort")) mask |= 2;
            if (strstr(e, "dsort")) mask |= 4;
            if (strstr(e, "emit")) mask |= 8;
            if (strstr(e, "project")) mask |= 16;
        }
        init = 1;
    }
    return mask;
}

// exact order among ties of the truncated depth key (2 launches)
static void launch_tie_fixup(RenderWork* w, cudaStream_t s) {
    depth_tie_fixup<<<148 * 4, kTieThreads, 0, s>>>(w->tkey[0], w->tkey[1], w->didx[0], w->didx[1], w->dkey[0],
                                                     w->ctr, w->tie_runs, w->dkey[1], w->tval[0], w->tie_k,
                                                     w->tval[1]);
}

// Enqueue one frame.  `project` enqueues the projection kernel into w.
template <class Proj>
static int render_enqueue(int64_t n, const CamDev& cam, RenderWork* w, Proj project,
                          float* out_rgb, uint8_t* out_rgb8, cudaStream_t s, bool readback = true) {
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    const int ntiles = ntx * nty;
    const int64_t npix = (int64_t)cam.width * cam.height;
    if (cam.width > 65535 || cam.height > 65535) return fail(GSV_E_INVALID_INPUT, "image too large");
    int rc = work_reserve(w, n, std::max<int64_t>(w->cap_k, 4 * n), ntiles, npix);
    if (rc) return rc;
    unsigned long long* ctr = w->ctr;
    int* npass = reinterpret_cast<int*>(ctr + C_NPASS);
    const SortScratch sc = sort_scratch(w);
    prof_mark(ST_PROJECT, s);
    reset_frame_kernel<<<1, 256, 0, s>>>(ctr, (long long)n, sc.ghist, reinterpret_cast<uint32_t*>(w->tile_done),
                                          ntiles, open_word(composite_rows()));
    const unsigned skip = debug_skip(), dbl = debug_double();
    if (!(skip & 16)) project();
    if (dbl & 16) {  // the second projection counts into spare counter slots
        unsigned long long* keep = w->ctr;
        w->ctr = keep + 16;
        project();
        w->ctr = keep;
    }
    count_launch(2);
    prof_mark(ST_DSORT, s);
    if (n > 0) {
        depth_key_prep<<<prep_grid(n), 256, 0, s>>>(w->dkey[0], w->tkey[0], ctr, sc.ghist, depth_key_bits());
        if (!(skip & 4))
            radix_sort<uint32_t>(w->tkey, w->didx, ctr + C_N, w->cap_n, depth_key_bits() / 8, npass, sc.ghist, sc, s);
        if (dbl & 4)
            radix_sort<uint32_t>(w->tkey, w->didx, ctr + C_N, w->cap_n, depth_key_bits() / 8, npass, sc.ghist, sc, s);
        launch_tie_fixup(w, s);
        if (dbl & 64) launch_tie_fixup(w, s);
        count_launch(2 + radix_launches(depth_key_bits() / 8, true));
    }
    prof_mark(ST_EMIT, s);
    std::vector<uint32_t> bounds;
    round_bounds(n, &bounds);
    const int tp = tile_passes(ntiles);
    for (size_t j = 0; j + 1 < bounds.size(); j++) {
        const uint32_t a = bounds[j], b = bounds[j + 1];
        prof_mark(ST_EMIT, s);
        const unsigned ge = std::max(1u, (unsigned)((b - a + kEmitTile - 1) / kEmitTile));
        uint32_t* th = sc.ghist + 1024 * (1 + (int)std::min<size_t>(j, kHistRegions - 2));
        uint32_t* mask = nullptr;  // first round: every tile open
        if (j > 0) {
            mask = w->open_mask;
            open_mask_kernel<<<(ntiles + 255) / 256, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(w->tile_done),
                                                                  ntiles, mask);
            count_launch(1);
        }
        // (binning needs the tile counters in shared memory and the tile scan
        // covers 32768 tiles: up to 4K frames; larger frames sort)
        const bool bin = r1_binning() && ntiles <= 32768 && (j == 0 || later_binning());
        const uint32_t* keys = w->tkey[tp & 1];
        const uint32_t* vals = w->tval[tp & 1];
        const uint32_t* toff = nullptr;
        if (bin) {
            // round 1: every tile open -> counting placement instead of emit + sort
            const uint32_t span = b - a;
            // rank blocks (at most 512): the placement walks a block
            // sequentially, the count matrix grows with the block count
            uint32_t B = std::max<uint32_t>(r1_block(), (span + 511u) / 512u);
            B = (B + 31u) & ~31u;
            const uint32_t nblk = std::max<uint32_t>(1u, (span + B - 1) / B);
            int rc = r1_reserve(w, (size_t)nblk * ntiles, (size_t)ntiles + 1);
            if (rc) return rc;
            const size_t sm = (size_t)ntiles * 4;
            if (int rc = r1_smem_attr(sm)) return rc;
            r1_count_kernel<<<nblk, 256, sm, s>>>(w->rect, w->didx[0], w->didx[1], ctr, a, b, B, ntx, ntiles, mask,
                                                  w->r1_bc);
            if (dbl & 256)
                r1_count_kernel<<<nblk, 256, sm, s>>>(w->rect, w->didx[0], w->didx[1], ctr, a, b, B, ntx, ntiles,
                                                      mask, w->r1_bc);
            r1_scan_blocks_kernel<<<(ntiles + 31) / 32, 32 * ((nblk + 31) / 32), 0, s>>>(w->r1_bc, (int)nblk, ntiles,
                                                                                          w->r1_off);
            r1_scan_tiles_kernel<<<1, 1024, 0, s>>>(w->r1_off, ntiles, ctr, (uint64_t)w->cap_k);
            prof_mark(ST_TSORT, s);
            launch_r1_place(nblk, sm, s, w->rect, w->didx[0], w->didx[1], ctr, a, b, B, ntx, ntiles, w->r1_bc,
                                                 w->r1_off, w->tval[0], (uint64_t)w->cap_k, mask);
            if (dbl & 512)
                launch_r1_place(nblk, sm, s, w->rect, w->didx[0], w->didx[1], ctr, a, b, B, ntx, ntiles, w->r1_bc,
                                                     w->r1_off, w->tval[0], (uint64_t)w->cap_k, mask);
            count_launch(4);
            keys = nullptr;
            vals = w->tval[0];
            toff = w->r1_off;
        } else {
            if (!(skip & 8))
                round_emit_fused<<<ge, kEmitThreads, 0, s>>>(w->rect, w->didx[0], w->didx[1], ctr, a, b, mask, ntiles,
                                                           w->tkey[0], w->tval[0], (uint64_t)w->cap_k, ntx, w->status,
                                                           w->ticket, ++w->epoch, th, tp);
            count_launch(1);
            prof_mark(ST_TSORT, s);
            if (!(skip & 2)) radix_sort<uint32_t>(w->tkey, w->tval, ctr + C_KCLAMP, w->cap_k, tp, nullptr, th, sc, s);
            if (dbl & 2) radix_sort<uint32_t>(w->tkey, w->tval, ctr + C_KCLAMP, w->cap_k, tp, nullptr, th, sc, s);
            count_launch(radix_launches(tp, true));
            if (later_ranges()) {  // tile ranges for the compositor instead of a key search per tile
                int rc = r1_reserve(w, 1, (size_t)ntiles + 1);
                if (rc) return rc;
                keys_to_off_kernel<<<148 * 2, 256, 0, s>>>(w->tkey[tp & 1], ctr, ntiles, w->r1_off);
                count_launch(1);
                toff = w->r1_off;
            }
        }
        prof_mark(ST_COMPOSITE, s);
        if ((dbl & 1) && j == 0)
            launch_composite_round(keys, toff, vals, ctr + C_KCLAMP, w->rec, w->state, w->tile_done, cam, true, false,
                                   out_rgb, out_rgb8, s);
        if (!(skip & 1))
            launch_composite_round(keys, toff, vals, ctr + C_KCLAMP, w->rec, w->state, w->tile_done, cam, j == 0,
                                   j + 2 == bounds.size(), out_rgb, out_rgb8, s);
        if ((dbl & 128) && j > 0 && j + 2 == bounds.size())
            launch_composite_round(keys, toff, vals, ctr + C_KCLAMP, w->rec, w->state, w->tile_done, cam, false, true,
                                   out_rgb, out_rgb8, s);
        count_launch(1);
    }
    prof_mark(ST_COUNT, s);
    // counters to the pinned mirror (a frame-parallel batch reads them back
    // once per stream at its end instead: the key-capacity maximum is sticky)
    if (readback) cudaMemcpyAsync(w->h_ctr, ctr, kCtrWords * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    GSV_CUDA(cudaGetLastError());
    return GSV_OK;
}

int readback_counters(RenderWork* w, cudaStream_t s) {
    if (!w->ctr) return GSV_OK;
    GSV_CUDA(cudaMemcpyAsync(w->h_ctr, w->ctr, kCtrWords * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    return GSV_OK;
}

// Enqueue, then check the key capacity; on overflow grow and re-render.
template <class Proj>
static int render_checked(int64_t n, const CamDev& cam, RenderWork* w, Proj project, float* out_rgb,
                          uint8_t* out_rgb8, gsv_render_stats* st, cudaStream_t s) {
    for (int attempt = 0; attempt < 6; attempt++) {
        int rc = render_enqueue(n, cam, w, project, out_rgb, out_rgb8, s);
        if (rc) return rc;
        GSV_CUDA(cudaStreamSynchronize(s));
        const unsigned long long K = w->h_ctr[C_MAXK];
        if (K <= (unsigned long long)w->cap_k) {
            if (st) {
                st->n_splats = n;
                st->n_visible = (int64_t)w->h_ctr[C_NVIS];
                st->n_keys = (int64_t)w->h_ctr[C_TOTK];
                st->n_keys_emitted = (int64_t)w->h_ctr[C_EMITK];
                st->tiles_x = (cam.width + kTile - 1) / kTile;
                st->tiles_y = (cam.height + kTile - 1) / kTile;
            }
            return GSV_OK;
        }
        rc = work_reserve(w, n, (int64_t)(K + K / 4 + 1024), 0, 0);
        if (rc) return rc;
    }
    return fail(GSV_E_NOMEM, "tile key buffer could not be sized");
}

int render_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
                  uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s) {
    const int64_t n = src.layer_off[src.nlayers];
    auto proj = [&]() { launch_project_planes(src, cam, w, s); };
    if (stats == reinterpret_cast<gsv_render_stats*>(1)) {  // enqueue only (throughput mode)
        return render_enqueue(n, cam, w, proj, out_rgb, out_rgb8, s, false);
    }
    return render_checked(n, cam, w, proj, out_rgb, out_rgb8, stats, s);
}

int render_soa(const SoaSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
               uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s) {
    auto proj = [&]() { launch_project_soa(src, cam, w, nullptr, nullptr, s); };
    return render_checked(src.n, cam, w, proj, out_rgb, out_rgb8, stats, s);
}

int render_splats2d(const Splat2DSrc& src, const CamDev& cam, RenderWork* w, float* out_rgb,
                    uint8_t* out_rgb8, gsv_render_stats* stats, cudaStream_t s) {
    auto proj = [&]() { launch_splat2d(src, cam, w, s); };
    return render_checked(src.n, cam, w, proj, out_rgb, out_rgb8, stats, s);
}

// ---------------------------------------------------------------------------
// psnr (metrics.py:31-38): the sum of squared differences on the device
// (fp64 accumulation); the host takes mean, log10 and the 99 dB cap.
template <typename T>
__global__ void sqdiff_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t n,
                              double* __restrict__ out) {
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = (double)a[i] - (double)b[i];
        acc = fma(d, d, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += ws[k];
        atomicAdd(out, t);
    }
}

void launch_sqdiff_f32(const float* a, const float* b, int64_t n, double* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(double), s);
    const int64_t g = std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (n > 0) sqdiff_kernel<float><<<(unsigned)std::max<int64_t>(g, 1), 256, 0, s>>>(a, b, n, out);
}

void launch_sqdiff_f64(const double* a, const double* b, int64_t n, double* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(double), s);
    const int64_t g = std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (n > 0) sqdiff_kernel<double><<<(unsigned)std::max<int64_t>(g, 1), 256, 0, s>>>(a, b, n, out);
}

// ---------------------------------------------------------------------------
// ssim (metrics.py:40-65): grayscale = channel mean, 11x11 Gaussian window
// (sigma 1.5, normalised) over valid positions, C1 = 0.01^2, C2 = 0.03^2,
// mean of the SSIM map.  The window is separable (outer product of the
// normalised 1-D Gaussian), so: gray -> horizontal 1-D pass of x, y, x^2,
// y^2, xy -> vertical pass + SSIM + block sums.  fp64 throughout.
__constant__ double c_g11[11];

template <typename T>
__global__ void ssim_gray(const T* __restrict__ a, const T* __restrict__ b, int64_t npix,
                          double* __restrict__ gx, double* __restrict__ gy) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
        gx[i] = (((double)a[3 * i] + (double)a[3 * i + 1]) + (double)a[3 * i + 2]) / 3.0;
        gy[i] = (((double)b[3 * i] + (double)b[3 * i + 1]) + (double)b[3 * i + 2]) / 3.0;
    }
}

__global__ void ssim_hpass(const double* __restrict__ gx, const double* __restrict__ gy, int H, int W,
                           double* __restrict__ h5) {
    const int Wv = W - 10;
    const int64_t n = (int64_t)H * Wv;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / Wv), j = (int)(o % Wv);
        const double* px = gx + (size_t)i * W + j;
        const double* py = gy + (size_t)i * W + j;
        double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int v = 0; v < 11; v++) {
            const double x = px[v], y = py[v], k = c_g11[v];
            s[0] = fma(k, x, s[0]);
            s[1] = fma(k, y, s[1]);
            s[2] = fma(k, x * x, s[2]);
            s[3] = fma(k, y * y, s[3]);
            s[4] = fma(k, x * y, s[4]);
        }
#pragma unroll
        for (int q = 0; q < 5; q++) h5[(size_t)q * n + o] = s[q];
    }
}

__global__ void ssim_vpass(const double* __restrict__ h5, int H, int W, double* __restrict__ total) {
    const int Wv = W - 10, Hv = H - 10;
    const int64_t n = (int64_t)H * Wv, nv = (int64_t)Hv * Wv;
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double acc = 0.0;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < nv; o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / Wv), j = (int)(o % Wv);
        double s[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 11; u++) {
            const size_t at = (size_t)(i + u) * Wv + j;
            const double k = c_g11[u];
#pragma unroll
            for (int q = 0; q < 5; q++) s[q] = fma(k, h5[(size_t)q * n + at], s[q]);
        }
        const double mx = s[0], my = s[1];
        const double vx = s[2] - mx * mx, vy = s[3] - my * my, cv = s[4] - mx * my;
        const double num = (2 * mx * my + C1) * (2 * cv + C2);
        const double den = (mx * mx + my * my + C1) * (vx + vy + C2);
        acc += num / den;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += ws[k];
        atomicAdd(total, t);
    }
}

int ssim_device(const void* a, const void* b, int H, int W, bool f64, double* out_mean, cudaStream_t s) {
    static bool init = false;
    if (!init) {  // _ssim_kernel (metrics.py:40-45), normalised 1-D factor
        double g[11], sum = 0;
        for (int v = 0; v < 11; v++) {
            const double x = v - 5.0;
            g[v] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
            sum += g[v];
        }
        for (int v = 0; v < 11; v++) g[v] /= sum;
        GSV_CUDA(cudaMemcpyToSymbol(c_g11, g, sizeof g));
        init = true;
    }
    const int64_t npix = (int64_t)H * W, nh = (int64_t)H * (W - 10);
    double* buf = nullptr;
    GSV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), (size_t)(2 * npix + 5 * nh + 1) * sizeof(double), s));
    double* gx = buf;
    double* gy = buf + npix;
    double* h5 = buf + 2 * npix;
    double* tot = h5 + 5 * nh;
    GSV_CUDA(cudaMemsetAsync(tot, 0, sizeof(double), s));
    const unsigned g = 148 * 8;
    if (f64) ssim_gray<double><<<g, 256, 0, s>>>(static_cast<const double*>(a), static_cast<const double*>(b), npix, gx, gy);
    else ssim_gray<float><<<g, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b), npix, gx, gy);
    ssim_hpass<<<g, 256, 0, s>>>(gx, gy, H, W, h5);
    ssim_vpass<<<g, 256, 0, s>>>(h5, H, W, tot);
    count_launch(3);
    double host = 0.0;
    GSV_CUDA(cudaMemcpyAsync(&host, tot, sizeof(double), cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaFreeAsync(buf, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    *out_mean = host / ((double)(H - 10) * (double)(W - 10));
    return GSV_OK;
}

__global__ void copy_order(const uint32_t* __restrict__ idx0, const uint32_t* __restrict__ idx1,
                           const unsigned long long* __restrict__ ctr, int32_t* __restrict__ order,
                           const SplatRec* __restrict__ rec, int32_t* __restrict__ tile_count) {
    const uint64_t n = ctr[C_N];
    const uint32_t nvis = (uint32_t)ctr[C_NVIS];
    const int np = reinterpret_cast<const int*>(ctr + C_NPASS)[0];
    const uint32_t* idx = (np & 1) ? idx1 : idx0;
    for (uint64_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const uint32_t i = idx[r];
        order[r] = (int32_t)i;
        if (tile_count) tile_count[i] = r < nvis ? (int32_t)rec_tile_count(rec[i]) : 0;
    }
}

// Projection outputs of one splat source for parity tests: rects, fp64
// depth, the stable depth order and per-splat tile counts, through the same
// projection and depth-sort kernels as a render.
template <class Proj>
static int project_debug_impl(int64_t n, RenderWork* w, Proj project, int32_t* order, int32_t* tile_count,
                              int64_t* n_visible, cudaStream_t s) {
    int rc = work_reserve(w, n, std::max<int64_t>(w->cap_k, n), 1, 0);
    if (rc) return rc;
    unsigned long long* ctr = w->ctr;
    int* npass = reinterpret_cast<int*>(ctr + C_NPASS);
    const SortScratch sc = sort_scratch(w);
    reset_frame_kernel<<<1, 256, 0, s>>>(ctr, (long long)n, sc.ghist, reinterpret_cast<uint32_t*>(w->tile_done), 0,
                                          0u);
    project();
    if (n > 0) {
        depth_key_prep<<<prep_grid(n), 256, 0, s>>>(w->dkey[0], w->tkey[0], ctr, sc.ghist, depth_key_bits());
        radix_sort<uint32_t>(w->tkey, w->didx, ctr + C_N, w->cap_n, depth_key_bits() / 8, npass, sc.ghist, sc, s);
        launch_tie_fixup(w, s);
        copy_order<<<148 * 4, 256, 0, s>>>(w->didx[0], w->didx[1], ctr, order, w->rec, tile_count);
    }
    cudaMemcpyAsync(w->h_ctr, ctr, kCtrWords * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    GSV_CUDA(cudaStreamSynchronize(s));
    GSV_CUDA(cudaGetLastError());
    if (n_visible) *n_visible = (int64_t)w->h_ctr[C_NVIS];
    return GSV_OK;
}

int project_debug(const SoaSrc& src, const CamDev& cam, RenderWork* w, int32_t* rects,
                  double* depth, int32_t* order, int32_t* tile_count, int64_t* n_visible,
                  cudaStream_t s) {
    // the rects and depths are only needed until the work buffers are sized
    int rc = work_reserve(w, src.n, std::max<int64_t>(w->cap_k, src.n), 1, 0);
    if (rc) return rc;
    return project_debug_impl(src.n, w, [&]() { launch_project_soa(src, cam, w, rects, depth, s); }, order,
                              tile_count, n_visible, s);
}

int project_debug_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, int32_t* rects,
                         double* depth, int32_t* order, int32_t* tile_count, int64_t* n_visible,
                         cudaStream_t s) {
    const int64_t n = src.layer_off[src.nlayers];
    return project_debug_impl(n, w, [&]() { launch_project_planes(src, cam, w, s, rects, depth); }, order,
                              tile_count, n_visible, s);
}

}  // namespace gsv
