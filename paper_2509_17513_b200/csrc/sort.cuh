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
template <typename K>
void radix_sort(K* keys[2], uint32_t* vals[2], const unsigned long long* n_ptr, int64_t cap,
                int npasses_max, const int* npasses_dev, uint32_t* hist, uint32_t* digit_total,
                cudaStream_t s);
int64_t radix_hist_words(int64_t cap);

// In-place exclusive scan of *n_ptr u32 counts; total -> *total_out.
void exclusive_scan(uint32_t* a, const unsigned long long* n_ptr, int64_t cap, uint32_t* bsum,
                    unsigned long long* total_out, cudaStream_t s);
int64_t scan_bsum_words(int64_t cap);

}  // namespace gsv
