// Device-wide stable LSD radix sort (8-bit digits) and exclusive scan.
//
// Element counts are read from device memory so a whole frame can be
// enqueued (and graph-captured) without a host round trip; grids are sized
// for the workspace capacity and blocks past the live count exit at once.
//
// One pass = upsweep (per-tile digit histograms) -> per-digit scan across
// tiles -> downsweep (stable scatter).  Stability inside a tile comes from
// processing the tile in index order, 256 items per round, with
// __match_any_sync giving each key its rank among same-digit keys of its
// warp and a per-warp/per-digit prefix giving the rank across warps.
#include <stdint.h>

#include "gsv_internal.h"
#include "sort.cuh"

namespace gsv {

constexpr int kRadix = 256;
constexpr int kThreads = 256;
constexpr int kRounds = 2;
constexpr int kTileItems = kThreads * kRounds;  // 2048

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) radix_upsweep(const K* __restrict__ keys,
                                                          const unsigned long long* __restrict__ n_ptr,
                                                          int shift, uint32_t* __restrict__ hist,
                                                          const int* __restrict__ npasses, int pass) {
    if (npasses && pass >= *npasses) return;
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kTileItems - 1) / kTileItems;
    __shared__ uint32_t cnt[kRadix];
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        cnt[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t base = b * kTileItems;
#pragma unroll
        for (int r = 0; r < kRounds; r++) {
            const uint32_t idx = base + r * kThreads + threadIdx.x;
            if (idx < n) atomicAdd(&cnt[(uint32_t)(keys[idx] >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        hist[(size_t)threadIdx.x * nb + b] = cnt[threadIdx.x];
        __syncthreads();
    }
}

// block d: exclusive scan of hist[d][0..nb) in place, total to digit_total[d]
__global__ void __launch_bounds__(kThreads) radix_scan(uint32_t* __restrict__ hist,
                                                       const unsigned long long* __restrict__ n_ptr,
                                                       uint32_t* __restrict__ digit_total,
                                                       const int* __restrict__ npasses, int pass) {
    if (npasses && pass >= *npasses) return;
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kTileItems - 1) / kTileItems;
    uint32_t* row = hist + (size_t)blockIdx.x * nb;
    __shared__ uint32_t warp_sum[kThreads / 32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c = 0; c < nb; c += kThreads) {
        const uint32_t i = c + threadIdx.x;
        const uint32_t v = i < nb ? row[i] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sum[warp] = x;
        __syncthreads();
        uint32_t wbase = 0;
        for (int w = 0; w < warp; w++) wbase += warp_sum[w];
        uint32_t total = 0;
        for (int w = 0; w < kThreads / 32; w++) total += warp_sum[w];
        const uint32_t cbase = carry;
        if (i < nb) row[i] = cbase + wbase + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = cbase + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) digit_total[blockIdx.x] = carry;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) radix_downsweep(const K* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin,
                                                            K* __restrict__ kout,
                                                            uint32_t* __restrict__ vout,
                                                            const unsigned long long* __restrict__ n_ptr,
                                                            int shift, const uint32_t* __restrict__ hist,
                                                            const uint32_t* __restrict__ digit_total,
                                                            const int* __restrict__ npasses, int pass) {
    if (npasses && pass >= *npasses) return;
    const uint32_t n = (uint32_t)*n_ptr;
    const uint32_t nb = (n + kTileItems - 1) / kTileItems;
    __shared__ uint32_t digit_base[kRadix];
    __shared__ uint32_t base[kRadix];
    __shared__ uint32_t wcnt[kThreads / 32][kRadix];
    __shared__ uint32_t wsum[kThreads / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    {  // exclusive scan of the digit totals
        const uint32_t v = digit_total[t];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t wb = 0;
        for (int w = 0; w < warp; w++) wb += wsum[w];
        digit_base[t] = wb + x - v;
        __syncthreads();
    }
    const uint32_t lt = lanemask_lt();
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        base[t] = digit_base[t] + hist[(size_t)t * nb + b];
        for (int r = 0; r < kRounds; r++) {
            const uint32_t idx = b * kTileItems + r * kThreads + t;
            const bool valid = idx < n;
            K k = 0;
            uint32_t v = 0, d = kRadix;
            if (valid) {
                k = kin[idx];
                v = vin[idx];
                d = (uint32_t)(k >> shift) & 0xFFu;
            }
#pragma unroll
            for (int w = 0; w < kThreads / 32; w++) wcnt[w][t] = 0;
            __syncthreads();
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t rank = __popc(peers & lt);
            if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
            __syncthreads();
            {
                uint32_t run = base[t];
#pragma unroll
                for (int w = 0; w < kThreads / 32; w++) {
                    const uint32_t c = wcnt[w][t];
                    wcnt[w][t] = run;
                    run += c;
                }
                base[t] = run;
            }
            __syncthreads();
            if (valid) {
                const uint32_t pos = wcnt[warp][d] + rank;
                kout[pos] = k;
                vout[pos] = v;
            }
            __syncthreads();
        }
    }
}

template <typename K>
void radix_sort(K* keys[2], uint32_t* vals[2], const unsigned long long* n_ptr, int64_t cap,
                int npasses_max, const int* npasses_dev, uint32_t* hist, uint32_t* digit_total,
                cudaStream_t s) {
    const int64_t tiles = (cap + kTileItems - 1) / kTileItems;
    const unsigned grid = (unsigned)(tiles < 148 * 8 ? (tiles > 0 ? tiles : 1) : 148 * 8);
    for (int p = 0; p < npasses_max; p++) {
        const int src = p & 1, dst = src ^ 1;
        radix_upsweep<K><<<grid, kThreads, 0, s>>>(keys[src], n_ptr, 8 * p, hist, npasses_dev, p);
        radix_scan<<<kRadix, kThreads, 0, s>>>(hist, n_ptr, digit_total, npasses_dev, p);
        radix_downsweep<K><<<grid, kThreads, 0, s>>>(keys[src], vals[src], keys[dst], vals[dst], n_ptr,
                                                     8 * p, hist, digit_total, npasses_dev, p);
    }
}

template void radix_sort<uint32_t>(uint32_t* [2], uint32_t* [2], const unsigned long long*, int64_t, int,
                                   const int*, uint32_t*, uint32_t*, cudaStream_t);
template void radix_sort<uint64_t>(uint64_t* [2], uint32_t* [2], const unsigned long long*, int64_t, int,
                                   const int*, uint32_t*, uint32_t*, cudaStream_t);

int64_t radix_hist_words(int64_t cap) {
    return (int64_t)kRadix * ((cap + kTileItems - 1) / kTileItems) + kRadix;
}

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
