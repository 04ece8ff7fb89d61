// Decode kernels: CRC-32 validation of every run and fp64 dequantization
// (the range decoder lives in rc_decode.cu).
//
// Compiled with -fmad=false: dequantize_codes (quantize.py:114-117) must not
// contract `rmin + code/top*(rmax-rmin)` into an FMA to stay bit-exact.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

// ---------------------------------------------------------------------------
// CRC-32 of every run (codec.py:260-262): the run's planes are split into
// kCrcChunk-byte chunks; each thread computes a chunk's standard CRC, shifts
// it by the bytes that follow it in the run (multiplication by x^(8*after)
// mod P: zlib's crc32_combine, applied to every chunk at once), and XORs it
// into the run accumulator.  XOR is commutative, so the result is
// deterministic.
//
// HBM-bound by design: a thread reads its 4 KiB chunk with 256-bit loads
// (every load instruction moves 32 full sectors), four loads in flight.  The
// byte tables are slicing-by-4 in shared memory replicated per lane -- entry
// (t, b) of lane l at word ((t * 256 + b) * 32 + l) -- so each lookup hits the
// lane's own bank (no conflicts for any data); 128 KiB per CTA, one CTA of
// 1024 threads per SM.
// ---------------------------------------------------------------------------
constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kCrcThreads = 1024;
constexpr size_t kCrcSmem = 4 * 256 * 32 * sizeof(uint32_t);
__constant__ uint32_t c_x2n[32];

__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

__device__ __forceinline__ uint32_t x8nmodp(uint64_t n) {  // x^(8n) mod P
    uint32_t p = 1u << 31;
    int k = 3;
    while (n) {
        if (n & 1) p = multmodp(c_x2n[k & 31], p);
        n >>= 1;
        k++;
    }
    return p;
}

// one table word of lane `lo` (= lane * 4 + table base): byte b of table t
__device__ __forceinline__ uint32_t tab(uint32_t lo, uint32_t t, uint32_t b) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(lo + (t * 256u + b) * 128u));
    return v;
}
// four bytes through the slicing-by-4 tables
__device__ __forceinline__ uint32_t crc_word(uint32_t lo, uint32_t crc, uint32_t w) {
    const uint32_t a = crc ^ w;
    return tab(lo, 3, a & 0xFFu) ^ tab(lo, 2, (a >> 8) & 0xFFu) ^ tab(lo, 1, (a >> 16) & 0xFFu) ^ tab(lo, 0, a >> 24);
}
__device__ __forceinline__ uint32_t crc_byte(uint32_t lo, uint32_t crc, uint32_t b) {
    return tab(lo, 0, (crc ^ b) & 0xFFu) ^ (crc >> 8);
}
struct U8x32 {
    uint32_t w[8];
};
__device__ __forceinline__ U8x32 ld256(const uint8_t* p) {
    U8x32 v;
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                   "=r"(v.w[7])
                 : "l"(p));
    return v;
}

__global__ void __launch_bounds__(kCrcThreads, 1) crc_kernel(const RunDesc* __restrict__ runs,
                                                             const PlaneRef* __restrict__ planes, int nplanes,
                                                             const uint32_t* __restrict__ chunk_prefix,
                                                             uint32_t nchunks, uint32_t* __restrict__ run_crc) {
    extern __shared__ __align__(16) uint32_t T[];  // [4][256][32]
    for (uint32_t i = threadIdx.x; i < 1024u; i += blockDim.x) {
        const uint32_t t = i >> 8, b = i & 255u;
        uint32_t c = b;  // byte b followed by t zero bytes
        for (uint32_t k = 0; k < 8u * (t + 1u); k++) c = (c & 1u) ? (kPoly ^ (c >> 1)) : (c >> 1);
        for (int l = 0; l < 32; l++) T[i * 32u + l] = c;
    }
    __syncthreads();
    const uint32_t lo = (uint32_t)__cvta_generic_to_shared(T) + 4u * (threadIdx.x & 31u);
    for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks; ch += gridDim.x * blockDim.x) {
        // plane of this chunk: last p with chunk_prefix[p] <= ch
        int plo = 0, phi = nplanes;
        while (phi - plo > 1) {
            const int mid = (plo + phi) >> 1;
            if (__ldg(chunk_prefix + mid) <= ch) plo = mid;
            else phi = mid;
        }
        const PlaneRef pr = planes[plo];
        const RunDesc r = runs[pr.run];
        const uint32_t off = (ch - __ldg(chunk_prefix + plo)) * kCrcChunk;
        const uint32_t len = min(kCrcChunk, r.plane_bytes - off);
        const uint8_t* p = pr.samples + off;
        uint32_t crc = 0xFFFFFFFFu;
        uint32_t i = 0;
        // bytes up to 32-B alignment (raw planes are consumed in place and may
        // start anywhere)
        const uint32_t head = min(len, (uint32_t)((32 - ((uintptr_t)p & 31)) & 31));
        for (; i < head; i++) crc = crc_byte(lo, crc, p[i]);
        // 128 B per step: four 256-bit loads issued before the tables run
        for (; i + 128 <= len; i += 128) {
            U8x32 v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = ld256(p + i + 32 * q);
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int k = 0; k < 8; k++) crc = crc_word(lo, crc, v[q].w[k]);
        }
        for (; i + 32 <= len; i += 32) {
            const U8x32 v = ld256(p + i);
#pragma unroll
            for (int k = 0; k < 8; k++) crc = crc_word(lo, crc, v.w[k]);
        }
        for (; i < len; i++) crc = crc_byte(lo, crc, p[i]);
        crc = ~crc;
        const uint64_t after = (uint64_t)(r.count - 1 - pr.f) * r.plane_bytes + (r.plane_bytes - off - len);
        if (after) crc = multmodp(x8nmodp(after), crc);
        atomicXor(run_crc + pr.run, crc);
    }
}

static void init_x2n_table() {
    static bool done = false;
    if (done) return;
    uint32_t tab[32];
    auto mm = [](uint32_t a, uint32_t b) {
        uint32_t m = 1u << 31, p = 0;
        for (;;) {
            if (a & m) {
                p ^= b;
                if ((a & (m - 1)) == 0) break;
            }
            m >>= 1;
            b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
        }
        return p;
    };
    uint32_t p = 1u << 30;  // x^1
    tab[0] = p;
    for (int n = 1; n < 32; n++) tab[n] = p = mm(p, p);
    cudaMemcpyToSymbol(c_x2n, tab, sizeof tab);
    done = true;
}

void launch_crc(const RunDesc* runs, const PlaneRef* planes, int nplanes,
                const uint32_t* chunk_prefix, uint32_t nchunks, uint32_t* run_crc,
                cudaStream_t s) {
    init_x2n_table();
    if (nchunks == 0) return;
    // the dynamic shared-memory limit is per device; setting it is cheap and
    // this runs once per container open
    cudaFuncSetAttribute(crc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrcSmem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t blocks = (nchunks + kCrcThreads - 1) / kCrcThreads;
    if (blocks > (uint32_t)sms) blocks = (uint32_t)sms;  // persistent: one CTA per SM
    crc_kernel<<<blocks, kCrcThreads, kCrcSmem, s>>>(runs, planes, nplanes, chunk_prefix, nchunks, run_crc);
}

// ---------------------------------------------------------------------------
// Dequantization (quantize.py:114-117) straight from the planes, and the
// frame assembly of _assemble_frames (container.py:229-257).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t load_sample(const uint8_t* p, uint32_t j, int bits) {
    if (bits == 8) return __ldg(p + j);
    if (bits == 16) {
        const uint8_t* q = p + 2 * (size_t)j;
        return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8);
    }
    const uint8_t* q = p + 4 * (size_t)j;
    return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16) |
           ((uint32_t)__ldg(q + 3) << 24);
}

__device__ __forceinline__ double dequant(uint32_t code, const SlotDesc& sd) {
    const double top = sd.dir_bits >= 32 ? 4294967295.0 : (double)((1ull << sd.dir_bits) - 1ull);
    return __dadd_rn(sd.rmin, __dmul_rn(__ddiv_rn((double)code, top), sd.span));
}

__global__ void dequant_frame_kernel(FrameSrc src, double* __restrict__ pos, double* __restrict__ rot,
                                     double* __restrict__ scl, double* __restrict__ opac,
                                     double* __restrict__ sh) {
    const int l = blockIdx.y;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n_l = src.layer_off[l + 1] - src.layer_off[l];
    if (j >= n_l) return;
    const uint32_t i = src.layer_off[l] + j;
    const int shdim = src.nslots - 11;
    const SlotDesc* sd = src.slots + (size_t)l * src.nslots;
    for (int s = 0; s < src.nslots; s++) {
        const SlotDesc d = sd[s];
        const double v = dequant(load_sample(d.samples, j, d.bits), d);
        if (s < 3) pos[3 * (size_t)i + s] = v;
        else if (s < 7) rot[4 * (size_t)i + (s - 3)] = v;
        else if (s < 10) scl[3 * (size_t)i + (s - 7)] = v;
        else if (s == 10) opac[i] = v;
        else sh[(size_t)shdim * i + (s - 11)] = v;
    }
}

void launch_dequant_frame(const FrameSrc& src, double* pos, double* rot, double* scl,
                          double* opac, double* sh, cudaStream_t s) {
    uint32_t maxn = 0;
    for (int l = 0; l < src.nlayers; l++) maxn = max(maxn, src.layer_off[l + 1] - src.layer_off[l]);
    if (maxn == 0) return;
    dim3 grid((maxn + 255) / 256, src.nlayers);
    dequant_frame_kernel<<<grid, 256, 0, s>>>(src, pos, rot, scl, opac, sh);
}

__global__ void frame_codes_kernel(FrameSrc src, uint32_t* __restrict__ out) {
    const int l = blockIdx.y;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n_l = src.layer_off[l + 1] - src.layer_off[l];
    if (j >= n_l) return;
    const uint32_t i = src.layer_off[l] + j;
    const SlotDesc* sd = src.slots + (size_t)l * src.nslots;
    for (int s = 0; s < src.nslots; s++) {
        out[(size_t)i * src.nslots + s] = load_sample(sd[s].samples, j, sd[s].bits);
    }
}

void launch_frame_codes(const FrameSrc& src, uint32_t* out, cudaStream_t s) {
    uint32_t maxn = 0;
    for (int l = 0; l < src.nlayers; l++) maxn = max(maxn, src.layer_off[l + 1] - src.layer_off[l]);
    if (maxn == 0) return;
    dim3 grid((maxn + 255) / 256, src.nlayers);
    frame_codes_kernel<<<grid, 256, 0, s>>>(src, out);
}

}  // namespace gsv

// ---------------------------------------------------------------------------
// Dev probe (tools/e2e_probe.py): a host-to-device copy done by SMs reading
// pinned host memory (UVA) with streaming (evict-first) stores, to measure
// whether the copy engine's writes through L2 slow the renders beside them.
// ---------------------------------------------------------------------------
namespace gsv {
__global__ void h2d_stream_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) v[k] = src[i + k * stride];
#pragma unroll
        for (int k = 0; k < 4; k++) __stcs(dst + i + k * stride, v[k]);
    }
    for (; i < n16; i += stride) __stcs(dst + i, src[i]);
}
}  // namespace gsv

extern "C" int gsv_dev_copy_h2d_stream(void* dst, const void* src, size_t n, void* stream, int blocks) {
    const size_t n16 = n / 16;
    if (n16)
        gsv::h2d_stream_kernel<<<blocks > 0 ? blocks : 148, 256, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), n16);
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
