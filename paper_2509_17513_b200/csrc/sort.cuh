// Declarations for sort.cu (device-count radix sort and scan).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gsv {

// Stable LSD radix sort of (keys, vals) over *n_ptr items.  keys[0]/vals[0]
// hold the input; after pass p the data is in buffer (p+1)&1.  When
// npasses_dev != nullptr, passes >= *npasses_dev are skipped on the device,
// so the result lives in buffer (*npasses_dev)&1; otherwise in
// npasses_max&1.
// Scratch of one stream's sorts: global digit histograms (4 x 256 u32),
// look-back status words (radix_status_words(cap) u64), a ticket counter and
// the host-side epoch that tags the status words of each pass.
struct SortScratch {
    uint32_t* ghist;
    unsigned long long* status;
    unsigned int* ticket;
    uint32_t* epoch;
};
// ghist: the keys' digit histograms (4 x 256 u32, byte p of the key in row
// p) already accumulated by the kernel that produced them, or nullptr to
// compute them here (one extra kernel).
template <typename K>
void radix_sort(K* keys[2], uint32_t* vals[2], const unsigned long long* n_ptr, int64_t cap,
                int npasses_max, const int* npasses_dev, uint32_t* ghist, const SortScratch& sc,
                cudaStream_t s);
int64_t radix_status_words(int64_t cap);
int radix_launches(int npasses, bool fused_hist);  // kernel launches of one radix_sort call

// In-place exclusive scan of *n_ptr u32 counts; total -> *total_out.
void exclusive_scan(uint32_t* a, const unsigned long long* n_ptr, int64_t cap, uint32_t* bsum,
                    unsigned long long* total_out, cudaStream_t s);
int64_t scan_bsum_words(int64_t cap);

}  // namespace gsv
