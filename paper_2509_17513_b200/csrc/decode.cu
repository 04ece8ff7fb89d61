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
// 1 KiB chunks; each thread computes a chunk's standard CRC with
// slicing-by-8 tables in shared memory, shifts it by the bytes that follow it
// in the run (multiplication by x^(8*after) mod P), and XORs it into the run
// accumulator.  XOR is commutative, so the result is deterministic.
// ---------------------------------------------------------------------------
constexpr uint32_t kCrcChunk = 1024;
constexpr uint32_t kPoly = 0xEDB88320u;
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

__global__ void __launch_bounds__(256) crc_kernel(const RunDesc* __restrict__ runs,
                                                  const PlaneRef* __restrict__ planes, int nplanes,
                                                  const uint32_t* __restrict__ chunk_prefix,
                                                  uint32_t nchunks, uint32_t* __restrict__ run_crc) {
    __shared__ uint32_t T[8][256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? (kPoly ^ (c >> 1)) : (c >> 1);
        T[0][i] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[0][i];
        for (int k = 1; k < 8; k++) {
            c = (c >> 8) ^ T[0][c & 0xFF];
            T[k][i] = c;
        }
    }
    __syncthreads();
    for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks;
         ch += gridDim.x * blockDim.x) {
        // plane of this chunk: last p with chunk_prefix[p] <= ch
        int lo = 0, hi = nplanes;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (chunk_prefix[mid] <= ch) lo = mid; else hi = mid;
        }
        const PlaneRef pr = planes[lo];
        const RunDesc r = runs[pr.run];
        const uint32_t off = (ch - chunk_prefix[lo]) * kCrcChunk;
        const uint32_t len = min(kCrcChunk, r.plane_bytes - off);
        const uint8_t* p = pr.samples + off;
        uint32_t crc = 0xFFFFFFFFu;
        uint32_t i = 0;
        // 16-B loads (a thread walks its own 1 KiB chunk, so every load
        // instruction touches 32 separate sectors: use all 16 B of each)
        const uint32_t head = (uint32_t)((16 - ((uintptr_t)p & 15)) & 15);
        for (; i < head && i < len; i++) crc = T[0][(crc ^ p[i]) & 0xFF] ^ (crc >> 8);
        for (; i + 16 <= len; i += 16) {
            const uint4 w = __ldcs(reinterpret_cast<const uint4*>(p + i));
            uint32_t a = crc ^ w.x, b = w.y;
            crc = T[7][a & 0xFF] ^ T[6][(a >> 8) & 0xFF] ^ T[5][(a >> 16) & 0xFF] ^ T[4][a >> 24] ^
                  T[3][b & 0xFF] ^ T[2][(b >> 8) & 0xFF] ^ T[1][(b >> 16) & 0xFF] ^ T[0][b >> 24];
            a = crc ^ w.z;
            b = w.w;
            crc = T[7][a & 0xFF] ^ T[6][(a >> 8) & 0xFF] ^ T[5][(a >> 16) & 0xFF] ^ T[4][a >> 24] ^
                  T[3][b & 0xFF] ^ T[2][(b >> 8) & 0xFF] ^ T[1][(b >> 16) & 0xFF] ^ T[0][b >> 24];
        }
        for (; i + 8 <= len; i += 8) {
            const uint2 w = *reinterpret_cast<const uint2*>(p + i);
            const uint32_t a = crc ^ w.x, b = w.y;
            crc = T[7][a & 0xFF] ^ T[6][(a >> 8) & 0xFF] ^ T[5][(a >> 16) & 0xFF] ^ T[4][a >> 24] ^
                  T[3][b & 0xFF] ^ T[2][(b >> 8) & 0xFF] ^ T[1][(b >> 16) & 0xFF] ^ T[0][b >> 24];
        }
        for (; i < len; i++) crc = T[0][(crc ^ p[i]) & 0xFF] ^ (crc >> 8);
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
    uint32_t blocks = (nchunks + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    crc_kernel<<<blocks, 256, 0, s>>>(runs, planes, nplanes, chunk_prefix, nchunks, run_crc);
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
