// Device-wide stable LSD radix sort (8-bit digits) and exclusive scan.
//
// Element counts are read from device memory so a whole frame can be
// enqueued (and graph-captured) without a host round trip; grids are sized
// for the workspace capacity and blocks past the live count exit at once.
//
// One histogram kernel for all passes, then one "onesweep" kernel per pass
// (tile-local ranking + decoupled look-back across tiles + scatter).
#include <stdint.h>

#include "gsv_internal.h"
#include "sort.cuh"

#include <algorithm>

namespace gsv {

constexpr int kRadix = 256;
constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileItems = kThreads * kItems;  // 2048 keys per CTA
constexpr int kMaxPasses = 4;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// All passes' global digit histograms in one read of the keys.
template <typename K>
__global__ void __launch_bounds__(kThreads) radix_hist(const K* __restrict__ keys,
                                                       const unsigned long long* __restrict__ n_ptr,
                                                       int npasses, uint32_t* __restrict__ ghist) {
    __shared__ uint32_t h[kMaxPasses][kRadix];
#pragma unroll
    for (int p = 0; p < kMaxPasses; p++) h[p][threadIdx.x] = 0;
    __syncthreads();
    const uint32_t n = (uint32_t)*n_ptr;
    for (uint32_t i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
        const K k = keys[i];
        for (int p = 0; p < npasses; p++) atomicAdd(&h[p][(uint32_t)(k >> (8 * p)) & 0xFFu], 1u);
    }
    __syncthreads();
    for (int p = 0; p < npasses; p++)
        if (h[p][threadIdx.x]) atomicAdd(&ghist[p * kRadix + threadIdx.x], h[p][threadIdx.x]);
}

__device__ __forceinline__ unsigned long long os_pack(uint32_t epoch, uint32_t flag, uint32_t v) {
    return ((unsigned long long)(epoch & 0xFFFFFFu) << 40) | ((unsigned long long)flag << 32) | v;
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// One stable LSD pass ("onesweep"): CTAs take tiles of 2048 keys in ticket
// order, rank their keys by digit locally (warp match + per-warp digit
// counts, in index order => stable), publish per-digit tile counts and
// resolve their global digit offsets with a decoupled look-back over the
// preceding tiles, then scatter.  One launch per pass, no host round trip.
template <typename K>
__global__ void __launch_bounds__(kThreads) radix_onesweep(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, const unsigned long long* __restrict__ n_ptr, int pass,
    const int* __restrict__ npasses, const uint32_t* __restrict__ ghist,
    unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket, uint32_t epoch) {
    if (npasses && pass >= *npasses) return;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wcnt[kThreads / 32][kRadix];
    __shared__ uint32_t s_dbase[kRadix];
    __shared__ uint32_t s_lbase[kRadix];
    __shared__ uint32_t s_wsum[kThreads / 32];
    __shared__ K s_k[kTileItems];
    __shared__ uint32_t s_v[kTileItems];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    // exclusive scan of this pass's global digit counts
    const uint32_t gv = ghist[pass * kRadix + t];
    uint32_t gx = gv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, gx, o);
        if (lane >= o) gx += y;
    }
    if (lane == 31) s_wsum[warp] = gx;
    __syncthreads();
    uint32_t gbase = gx - gv;
    for (int w = 0; w < warp; w++) gbase += s_wsum[w];
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t ntiles = (n + kTileItems - 1) / kTileItems;
    // persistent CTAs take tiles in ticket order until none is left; every
    // CTA ends with one ticket past the end, so the last of those resets
    for (;;) {
    __syncthreads();
    if (t == 0) {
        const uint32_t tk = atomicAdd(ticket, 1u);
        if (tk == ntiles + gridDim.x - 1) *ticket = 0;
        s_tile = tk;
    }
#pragma unroll
    for (int w = 0; w < kThreads / 32; w++) s_wcnt[w][t] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const int shift = 8 * pass;
    const uint32_t base = tile * kTileItems + warp * (32 * kItems) + lane;
    K k[kItems];
    uint32_t v[kItems], d[kItems], r[kItems];
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        const uint32_t idx = base + i * 32;
        const bool ok = idx < n;
        k[i] = ok ? kin[idx] : K(0);
        v[i] = ok ? vin[idx] : 0u;
        d[i] = ok ? ((uint32_t)(k[i] >> shift) & 0xFFu) : kRadix;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
        const uint32_t cnt = d[i] < kRadix ? s_wcnt[warp][d[i]] : 0u;
        r[i] = cnt + __popc(peers & lt);
        __syncwarp();
        if (d[i] < kRadix && (peers & lt) == 0) s_wcnt[warp][d[i]] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // digit t: offsets of each warp's run inside the tile, tile total
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; w++) {
        const uint32_t c = s_wcnt[w][t];
        s_wcnt[w][t] = tot;
        tot += c;
    }
    uint32_t prefix = 0;
    if (tile == 0) {
        atomicExch(status + t, os_pack(epoch, 2, tot));
    } else {
        atomicExch(status + (size_t)tile * kRadix + t, os_pack(epoch, 1, tot));
        // look back kLook tiles per step (independent loads), summing
        // aggregates up to the nearest inclusive prefix; an entry not yet
        // published ends the step and is re-read in the next one
        constexpr int kLook = 16;
        const uint32_t ep = epoch & 0xFFFFFFu;
        int j = (int)tile - 1;
        for (;;) {
            unsigned long long w[kLook];
#pragma unroll
            for (int q = 0; q < kLook; q++)
                w[q] = j - q >= 0 ? ld_volatile_u64(status + (size_t)(j - q) * kRadix + t) : 0ull;
            bool done = false;
            int q = 0;
#pragma unroll
            for (; q < kLook; q++) {
                const uint32_t fl = (uint32_t)(w[q] >> 32) & 0xFFu;
                if ((uint32_t)(w[q] >> 40) != ep || fl == 0) break;
                prefix += (uint32_t)w[q];
                if (fl == 2) {
                    done = true;
                    break;
                }
            }
            if (done) break;
            j -= q;
        }
        atomicExch(status + (size_t)tile * kRadix + t, os_pack(epoch, 2, prefix + tot));
    }
    s_dbase[t] = gbase + prefix;
    // tile-local digit bases (exclusive scan of the digit totals), then the
    // keys are staged in shared memory in digit order so the global writes of
    // each digit's run are coalesced
    uint32_t lx = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, lx, o);
        if (lane >= o) lx += y;
    }
    __syncthreads();  // s_wsum reuse
    if (lane == 31) s_wsum[warp] = lx;
    __syncthreads();
    uint32_t lb = lx - tot;
    for (int w = 0; w < warp; w++) lb += s_wsum[w];
    s_lbase[t] = lb;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        if (d[i] < kRadix) {
            const uint32_t lp = s_lbase[d[i]] + s_wcnt[warp][d[i]] + r[i];
            s_k[lp] = k[i];
            s_v[lp] = v[i];
        }
    }
    __syncthreads();
    const uint32_t valid = min((uint32_t)kTileItems, n - tile * kTileItems);
    for (uint32_t i = t; i < valid; i += kThreads) {
        const K key = s_k[i];
        const uint32_t dg = (uint32_t)(key >> shift) & 0xFFu;
        const uint32_t pos = s_dbase[dg] + (i - s_lbase[dg]);
        kout[pos] = key;
        vout[pos] = s_v[i];
    }
    }  // next tile
}

template <typename K>
void radix_sort(K* keys[2], uint32_t* vals[2], const unsigned long long* n_ptr, int64_t cap,
                int npasses_max, const int* npasses_dev, uint32_t* ghist, const SortScratch& sc,
                cudaStream_t s) {
    const int64_t tiles = (cap + kTileItems - 1) / kTileItems;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 2));
    if (!ghist) {  // histograms not provided by the producer of the keys
        ghist = sc.ghist;
        cudaMemsetAsync(ghist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s);
        const unsigned hgrid = (unsigned)std::min<int64_t>(std::max<int64_t>((cap + 4095) / 4096, 1), 148 * 2);
        radix_hist<K><<<hgrid, kThreads, 0, s>>>(keys[0], n_ptr, npasses_max, ghist);
    }
    for (int p = 0; p < npasses_max; p++) {
        const int src = p & 1, dst = src ^ 1;
        radix_onesweep<K><<<grid, kThreads, 0, s>>>(keys[src], vals[src], keys[dst], vals[dst], n_ptr, p,
                                                    npasses_dev, ghist, sc.status, sc.ticket, ++*sc.epoch);
    }
}

template void radix_sort<uint32_t>(uint32_t* [2], uint32_t* [2], const unsigned long long*, int64_t, int,
                                   const int*, uint32_t*, const SortScratch&, cudaStream_t);

int64_t radix_status_words(int64_t cap) { return (int64_t)kRadix * ((cap + kTileItems - 1) / kTileItems); }
int radix_launches(int npasses, bool fused_hist) { return (fused_hist ? 0 : 1) + npasses; }

// ---------------------------------------------------------------------------
// Exclusive scan of u32 counts in place; total -> *total_out (u64).
// ---------------------------------------------------------------------------
constexpr int kScanItems = kThreads * 8;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wsum, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    total = 0;
    for (int w = 0; w < kThreads / 32; w++) {
        if (w < warp) wb += wsum[w];
        total += wsum[w];
    }
    __syncthreads();
    return wb + x - v;
}

__global__ void __launch_bounds__(kThreads) scan_reduce(const uint32_t* __restrict__ a,
                                                        const unsigned long long* __restrict__ n_ptr,
                                                        uint32_t* __restrict__ bsum) {
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kScanItems - 1) / kScanItems;
    __shared__ uint32_t wsum[kThreads / 32];
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        uint32_t s = 0;
        const uint32_t base = b * kScanItems + threadIdx.x * 8;
#pragma unroll
        for (int k = 0; k < 8; k++) s += (base + k < n) ? a[base + k] : 0u;
        uint32_t total;
        block_excl_scan(s, wsum, total);
        if (threadIdx.x == 0) bsum[b] = total;
    }
}

__global__ void __launch_bounds__(1024) scan_bsums(uint32_t* __restrict__ bsum,
                                                   const unsigned long long* __restrict__ n_ptr,
                                                   unsigned long long* __restrict__ total_out) {
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kScanItems - 1) / kScanItems;
    __shared__ unsigned long long carry;
    __shared__ uint32_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c = 0; c < nb; c += 1024) {
        const uint32_t i = c + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t wb = 0, tot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wb += wsum[w];
            tot += wsum[w];
        }
        const unsigned long long cb = carry;
        if (i < nb) bsum[i] = (uint32_t)(cb + wb + x - v);
        __syncthreads();
        if (threadIdx.x == 0) carry = cb + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total_out = carry;
}

__global__ void __launch_bounds__(kThreads) scan_apply(uint32_t* __restrict__ a,
                                                       const unsigned long long* __restrict__ n_ptr,
                                                       const uint32_t* __restrict__ bsum) {
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kScanItems - 1) / kScanItems;
    __shared__ uint32_t wsum[kThreads / 32];
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const uint32_t base = b * kScanItems + threadIdx.x * 8;
        uint32_t v[8], s = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = (base + k < n) ? a[base + k] : 0u;
            s += v[k];
        }
        uint32_t total;
        uint32_t run = bsum[b] + block_excl_scan(s, wsum, total);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (base + k < n) a[base + k] = run;
            run += v[k];
        }
    }
}

void exclusive_scan(uint32_t* a, const unsigned long long* n_ptr, int64_t cap, uint32_t* bsum,
                    unsigned long long* total_out, cudaStream_t s) {
    const int64_t tiles = (cap + kScanItems - 1) / kScanItems;
    const unsigned grid = (unsigned)(tiles < 148 * 8 ? (tiles > 0 ? tiles : 1) : 148 * 8);
    scan_reduce<<<grid, kThreads, 0, s>>>(a, n_ptr, bsum);
    scan_bsums<<<1, 1024, 0, s>>>(bsum, n_ptr, total_out);
    scan_apply<<<grid, kThreads, 0, s>>>(a, n_ptr, bsum);
}

int64_t scan_bsum_words(int64_t cap) { return (cap + kScanItems - 1) / kScanItems + 1; }

}  // namespace gsv
