// EWA projection (render.py:185-287) fused with dequantization, SH colour,
// conic inversion (render.py:346-349) and record emission; plus the
// reconstruct_frame delta fold (motion.py:165-235).
//
// fp64 throughout and compiled with -fmad=false: the reference's order of
// operations is reproduced exactly, with __fma_rn exactly where numpy hands
// the work to OpenBLAS (x_cam = P @ R.T and the stacked 3x3 products were
// measured to be fma(a2,b2, fma(a1,b1, a0*b0)) chains).  Rects, culling,
// depth and therefore sort order are bit-identical to the reference.
#include <stdint.h>

#include "gsv_internal.h"

namespace gsv {

__device__ __forceinline__ double np_max(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b));
}
__device__ __forceinline__ double np_min(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b));
}

__device__ __forceinline__ uint32_t load_sample_p(const uint8_t* p, uint32_t j, int bits) {
    if (bits == 8) return __ldg(p + j);
    if (bits == 16) {
        const uint8_t* q = p + 2 * (size_t)j;
        return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8);
    }
    const uint8_t* q = p + 4 * (size_t)j;
    return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16) |
           ((uint32_t)__ldg(q + 3) << 24);
}

// code / (2^bits - 1) for 8- and 16-bit codes, tabulated: the quotient is the
// correctly rounded fp64 division, so rmin + q * (rmax - rmin) stays
// bit-identical to dequantize_codes (quantize.py:114-117) without an fp64
// division per channel.
__device__ double g_q8[256];
__device__ double g_q16[65536];

__device__ __forceinline__ double dequant_p(uint32_t code, const SlotDesc& sd) {
    double q;
    if (sd.dir_bits == 8 && code < 256u) q = __ldg(g_q8 + code);
    else if (sd.dir_bits == 16 && code < 65536u) q = __ldg(g_q16 + code);
    else q = __ddiv_rn((double)code, sd.dir_bits >= 32 ? 4294967295.0
                                                        : (double)((1ull << sd.dir_bits) - 1ull));
    return __dadd_rn(sd.rmin, __dmul_rn(q, sd.span));
}

static void init_quotient_tables() {
    static bool done = false;
    if (done) return;
    static double t8[256], t16[65536];
    for (int i = 0; i < 256; i++) t8[i] = (double)i / 255.0;
    for (int i = 0; i < 65536; i++) t16[i] = (double)i / 65535.0;
    cudaMemcpyToSymbol(g_q8, t8, sizeof t8);
    cudaMemcpyToSymbol(g_q16, t16, sizeof t16);
    done = true;
}

// Splat attributes in fp64 registers.
template <int DEG>
struct SplatIn {
    static constexpr int SHD = 3 * (DEG + 1) * (DEG + 1);
    double p[3], q[4], s[3], o;
    double sh[SHD];
};

// Samples of one slot: 16-bit samples are read with one aligned 16-bit load
// when the plane is 2-B aligned (codec-0 planes are consumed in place and
// may not be).
__device__ __forceinline__ uint32_t load_sample_fast(const uint8_t* p, uint32_t j, int bits) {
    if (bits == 8) return __ldg(p + j);
    if (bits == 16) {
        const uint8_t* q = p + 2 * (size_t)j;
        if ((reinterpret_cast<uintptr_t>(p) & 1u) == 0)
            return __ldg(reinterpret_cast<const uint16_t*>(q));
        return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8);
    }
    return load_sample_p(p, j, bits);
}

// Per block: the frame's slot descriptors and the 8-bit quotient table live in
// shared memory (stage() in the kernel prologue), so a slot costs one LDS
// for its descriptor and one global load for its code; all of a splat's
// codes are loaded before any is dequantized.
struct PlaneLoader {
    FrameSrc src;
    __device__ __forceinline__ int64_t count() const { return src.layer_off[src.nlayers]; }
    static size_t smem_bytes(const FrameSrc& f) { return 256 * sizeof(double) + (size_t)f.nlayers * f.nslots * sizeof(SlotDesc); }
    __device__ __forceinline__ void stage(unsigned char* smem) const {
        double* q8 = reinterpret_cast<double*>(smem);
        SlotDesc* sd = reinterpret_cast<SlotDesc*>(smem + 256 * sizeof(double));
        for (int k = threadIdx.x; k < 256; k += blockDim.x) q8[k] = g_q8[k];
        const int nsd = src.nlayers * src.nslots;
        for (int k = threadIdx.x; k < nsd; k += blockDim.x) sd[k] = src.slots[k];
        __syncthreads();
    }
    __device__ __forceinline__ double deq(uint32_t code, const SlotDesc& d, const double* s_q8) const {
        double q;
        if (d.dir_bits == 8 && code < 256u) q = s_q8[code];
        else if (d.dir_bits == 16 && code < 65536u) q = __ldg(g_q16 + code);
        else q = __ddiv_rn((double)code, d.dir_bits >= 32 ? 4294967295.0 : (double)((1ull << d.dir_bits) - 1ull));
        return __dadd_rn(d.rmin, __dmul_rn(q, d.span));
    }
    // Every code of the splat is fetched first (one round of independent
    // loads: the SH codes' latency overlaps the geometry's); geometry slots
    // (0..10) are dequantised before the projection, SH slots (11..) only
    // for survivors.
    template <int DEG>
    struct Codes {
        uint32_t c[11 + SplatIn<DEG>::SHD];
        int l;  // the splat's layer (found once, by fetch)
    };
    template <int DEG>
    __device__ __forceinline__ void fetch(uint32_t i, Codes<DEG>& k, const unsigned char* smem) const {
        const SlotDesc* s_sd = reinterpret_cast<const SlotDesc*>(smem + 256 * sizeof(double));
        int l = 0;
        while (l + 1 < src.nlayers && src.layer_off[l + 1] <= i) l++;
        k.l = l;
        const uint32_t j = i - src.layer_off[l];
        const SlotDesc* sd = s_sd + (size_t)l * src.nslots;
#pragma unroll
        for (int s = 0; s < 11 + SplatIn<DEG>::SHD; s++) k.c[s] = load_sample_fast(sd[s].samples, j, sd[s].bits);
    }
    template <int DEG, int S0, int S1>
    __device__ __forceinline__ void load(uint32_t i, const Codes<DEG>& k, SplatIn<DEG>& a,
                                         const unsigned char* smem) const {
        const double* s_q8 = reinterpret_cast<const double*>(smem);
        const SlotDesc* s_sd = reinterpret_cast<const SlotDesc*>(smem + 256 * sizeof(double));
        const SlotDesc* sd = s_sd + (size_t)k.l * src.nslots;
#pragma unroll
        for (int s = S0; s < S1; s++) {
            const double v = deq(k.c[s], sd[s], s_q8);
            if (s < 3) a.p[s] = v;
            else if (s < 7) a.q[s - 3] = v;
            else if (s < 10) a.s[s - 7] = v;
            else if (s == 10) a.o = v;
            else a.sh[s - 11] = v;
        }
    }
};

struct SoaLoader {
    SoaSrc src;
    static size_t smem_bytes(const SoaSrc&) { return 0; }
    __device__ __forceinline__ void stage(unsigned char*) const {}
    __device__ __forceinline__ int64_t count() const { return src.n; }
    template <int DEG>
    struct Codes {};
    template <int DEG>
    __device__ __forceinline__ void fetch(uint32_t, Codes<DEG>&, const unsigned char*) const {}
    template <int DEG, int S0, int S1>
    __device__ __forceinline__ void load(uint32_t i, const Codes<DEG>&, SplatIn<DEG>& a,
                                         const unsigned char*) const {
        constexpr int shdim = SplatIn<DEG>::SHD;
        if constexpr (S0 == 0) {
#pragma unroll
            for (int k = 0; k < 3; k++) a.p[k] = src.pos[3 * (size_t)i + k];
#pragma unroll
            for (int k = 0; k < 4; k++) a.q[k] = src.rot[4 * (size_t)i + k];
#pragma unroll
            for (int k = 0; k < 3; k++) a.s[k] = src.scl[3 * (size_t)i + k];
            a.o = src.opac[i];
        } else {
#pragma unroll
            for (int k = 0; k < shdim; k++) a.sh[k] = src.sh[(size_t)shdim * i + k];
        }
    }
};

__constant__ double c_sh2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
__constant__ double c_sh3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

// eval_sh_colors (render.py:202-237), same association order
template <int DEG>
__device__ __forceinline__ void sh_color(const SplatIn<DEG>& a, const CamDev& cam, double rgb[3]) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    double col[3];
    for (int c = 0; c < 3; c++) col[c] = C0 * a.sh[c];
    if constexpr (DEG >= 1) {
        const double dx = a.p[0] - cam.center[0], dy = a.p[1] - cam.center[1], dz = a.p[2] - cam.center[2];
        double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
        if (nrm == 0.0) nrm = 1.0;
        const double x = dx / nrm, y = dy / nrm, z = dz / nrm;
        for (int c = 0; c < 3; c++)
            col[c] = ((col[c] - (C1 * y) * a.sh[3 + c]) + (C1 * z) * a.sh[6 + c]) - (C1 * x) * a.sh[9 + c];
        if constexpr (DEG >= 2) {
            const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            for (int c = 0; c < 3; c++) {
                double v = col[c];
                v = v + (c_sh2[0] * xy) * a.sh[12 + c];
                v = v + (c_sh2[1] * yz) * a.sh[15 + c];
                v = v + (c_sh2[2] * ((2.0 * zz - xx) - yy)) * a.sh[18 + c];
                v = v + (c_sh2[3] * xz) * a.sh[21 + c];
                v = v + (c_sh2[4] * (xx - yy)) * a.sh[24 + c];
                col[c] = v;
            }
            if constexpr (DEG >= 3) {
                for (int c = 0; c < 3; c++) {
                    double v = col[c];
                    v = v + ((c_sh3[0] * y) * (3.0 * xx - yy)) * a.sh[27 + c];
                    v = v + ((c_sh3[1] * xy) * z) * a.sh[30 + c];
                    v = v + ((c_sh3[2] * y) * ((4.0 * zz - xx) - yy)) * a.sh[33 + c];
                    v = v + ((c_sh3[3] * z) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy)) * a.sh[36 + c];
                    v = v + ((c_sh3[4] * x) * ((4.0 * zz - xx) - yy)) * a.sh[39 + c];
                    v = v + ((c_sh3[5] * z) * (xx - yy)) * a.sh[42 + c];
                    v = v + ((c_sh3[6] * x) * (xx - 3.0 * yy)) * a.sh[45 + c];
                    col[c] = v;
                }
            }
        }
    }
    for (int c = 0; c < 3; c++) rgb[c] = np_min(np_max(col[c] + 0.5, 0.0), 1.0);
}

// 3x3 product as OpenBLAS evaluates it
__device__ __forceinline__ void mm3(const double* A, const double* B, double* C) {
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++)
            C[i * 3 + k] = __fma_rn(A[i * 3 + 2], B[6 + k], __fma_rn(A[i * 3 + 1], B[3 + k], A[i * 3] * B[k]));
}

struct ProjOut {
    bool alive;
    double depth;
    double u, v;
    double cov[4];
    double x0, x1, y0, y1;
};

// project_set for one splat (render.py:251-280)
template <int DEG>
__device__ __forceinline__ ProjOut project_one(const SplatIn<DEG>& a, const CamDev& cam) {
    ProjOut o;
    const double* R = cam.R;
    double cp[3];
#pragma unroll
    for (int r = 0; r < 3; r++)
        cp[r] = __fma_rn(R[r * 3 + 2], a.p[2], __fma_rn(R[r * 3 + 1], a.p[1], R[r * 3] * a.p[0])) + cam.t[r];
    o.depth = cp[2];
    bool al = cp[2] > cam.near_;
    // _quat_to_rotmats (render.py:185-199)
    const double qn = sqrt(((a.q[0] * a.q[0] + a.q[1] * a.q[1]) + a.q[2] * a.q[2]) + a.q[3] * a.q[3]);
    const double w = a.q[0] / qn, x = a.q[1] / qn, y = a.q[2] / qn, z = a.q[3] / qn;
    double m[9];
    m[0] = 1 - 2 * (y * y + z * z);
    m[1] = 2 * (x * y - w * z);
    m[2] = 2 * (x * z + w * y);
    m[3] = 2 * (x * y + w * z);
    m[4] = 1 - 2 * (x * x + z * z);
    m[5] = 2 * (y * z - w * x);
    m[6] = 2 * (x * z - w * y);
    m[7] = 2 * (y * z + w * x);
    m[8] = 1 - 2 * (x * x + y * y);
    const double s2[3] = {a.s[0] * a.s[0], a.s[1] * a.s[1], a.s[2] * a.s[2]};
    double cw[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++)
            cw[i * 3 + k] = ((m[i * 3] * s2[0]) * m[k * 3] + (m[i * 3 + 1] * s2[1]) * m[k * 3 + 1]) +
                            (m[i * 3 + 2] * s2[2]) * m[k * 3 + 2];
    double RT[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) RT[i * 3 + j] = R[j * 3 + i];
    double tmp[9], cc[9];
    mm3(R, cw, tmp);
    mm3(tmp, RT, cc);
    const double zz = al ? cp[2] : 1.0;
    o.u = cam.fx * cp[0] / zz + cam.cx;
    o.v = cam.fy * cp[1] / zz + cam.cy;
    const double J[6] = {cam.fx / zz, 0.0, -cam.fx * cp[0] / (zz * zz), 0.0, cam.fy / zz,
                         -cam.fy * cp[1] / (zz * zz)};
#pragma unroll
    for (int aa = 0; aa < 2; aa++)
#pragma unroll
        for (int d = 0; d < 2; d++) {
            double acc = (J[aa * 3] * cc[0]) * J[d * 3];
#pragma unroll
            for (int t = 1; t < 9; t++) {
                const int b = t / 3, c = t % 3;
                acc = acc + (J[aa * 3 + b] * cc[b * 3 + c]) * J[d * 3 + c];
            }
            o.cov[aa * 2 + d] = acc;
        }
    o.cov[0] += 0.3;
    o.cov[3] += 0.3;
    const double A = o.cov[0], B = o.cov[1], C = o.cov[3];
    const double hm = (A - C) / 2;
    const double lam = (A + C) / 2 + sqrt(hm * hm + B * B);
    const double radius = ceil(3.0 * sqrt(np_max(lam, 0.0)));
    o.x0 = np_max(floor(o.u - radius), 0.0);
    o.x1 = np_min(floor(o.u + radius) + 1, (double)cam.width);
    o.y0 = np_max(floor(o.v - radius), 0.0);
    o.y1 = np_min(floor(o.v + radius) + 1, (double)cam.height);
    o.alive = al && (o.x0 < o.x1) && (o.y0 < o.y1);
    return o;
}

// One thread per splat.  Writes the depth sort key (fp64 bits; culled splats
// get ~0 so they sort last), the splat index, and the 48-B record; counts
// survivors and tracks the depth-bit range of the survivors.
__device__ __forceinline__ uint32_t rect_tiles(uint32_t rx, uint32_t ry) {
    const uint32_t x0 = rx & 0xFFFFu, x1 = rx >> 16, y0 = ry & 0xFFFFu, y1 = ry >> 16;
    return ((x1 - 1) / kTile - x0 / kTile + 1) * ((y1 - 1) / kTile - y0 / kTile + 1);
}

template <class Loader, int DEG, int REGS = 80>
__global__ void __launch_bounds__(128) __maxnreg__(REGS) project_kernel(Loader ld, CamDev cam,
                                                      uint64_t* __restrict__ dkey,
                                                      uint32_t* __restrict__ didx,
                                                      SplatRec* __restrict__ rec,
                                                      uint2* __restrict__ rect,
                                                      unsigned long long* __restrict__ ctr,
                                                      int32_t* __restrict__ dbg_rect,
                                                      double* __restrict__ dbg_depth) {
    extern __shared__ __align__(16) unsigned char proj_smem[];
    ld.stage(proj_smem);
    const int64_t n = ld.count();
    // persistent CTAs (grid <= one wave): the slot descriptors and quotient
    // table are staged once per CTA, not once per 128 splats
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool alive = false;
    uint64_t key = ~0ull;
    uint32_t ntile = 0;  // (tile, splat) overlaps of this splat's rect (render stats)
    if (i < n) {
        SplatIn<DEG> a;
        typename Loader::template Codes<DEG> codes;
        ld.template fetch<DEG>((uint32_t)i, codes, proj_smem);
        ld.template load<DEG, 0, 11>((uint32_t)i, codes, a, proj_smem);
        const ProjOut o = project_one(a, cam);
        alive = o.alive;
        if (dbg_depth) dbg_depth[i] = o.depth;
        if (alive) {
            key = (uint64_t)__double_as_longlong(o.depth);
            ld.template load<DEG, 11, 11 + SplatIn<DEG>::SHD>((uint32_t)i, codes, a, proj_smem);
            double rgb[3];
            sh_color(a, cam, rgb);
            const double det = o.cov[0] * o.cov[3] - o.cov[1] * o.cov[1];
            SplatRec r;
            r.fx0 = (float)o.x0;
            r.fy0 = (float)o.y0;
            r.fx1 = (float)o.x1;
            r.fy1 = (float)o.y1;
            r.ox = (float)(o.u - o.x0);
            r.oy = (float)(o.v - o.y0);
            // conic (render.py:346-349) folded into the base-2 exponent the
            // compositor evaluates: log2(e) * -0.5 * (a dx^2 + 2 b dx dy + c dy^2)
            const double l2e = 1.4426950408889634;
            r.ca = (float)(-0.5 * l2e * (o.cov[3] / det));
            r.cb = (float)(-l2e * (-o.cov[1] / det));
            r.cc = (float)(-0.5 * l2e * (o.cov[0] / det));
            r.r = (float)rgb[0];
            r.g = (float)rgb[1];
            r.b = (float)rgb[2];
            r.op = (float)np_max(a.o, 0.0);  // alpha <= 0 draws nothing (render.py:326)
            r.pad = __float_as_uint(r.op > 0.f ? log2f(r.op) : -INFINITY);  // log2 op for the compositor
            r.rx = (uint32_t)o.x0 | ((uint32_t)o.x1 << 16);
            r.ry = (uint32_t)o.y0 | ((uint32_t)o.y1 << 16);
            rec[i] = r;
            rect[i] = make_uint2(r.rx, r.ry);
            ntile = rect_tiles(r.rx, r.ry);
        }
        if (dbg_rect) {
            dbg_rect[4 * i] = alive ? (int32_t)o.x0 : 0;
            dbg_rect[4 * i + 1] = alive ? (int32_t)o.x1 : 0;
            dbg_rect[4 * i + 2] = alive ? (int32_t)o.y0 : 0;
            dbg_rect[4 * i + 3] = alive ? (int32_t)o.y1 : 0;
        }
        dkey[i] = key;
        didx[i] = (uint32_t)i;
    }
    // warp-aggregated survivor count and depth-bit range
    const unsigned m = __ballot_sync(0xffffffffu, alive);
    uint64_t kmin = alive ? key : ~0ull, kmax = alive ? key : 0ull;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        kmin = min(kmin, (uint64_t)__shfl_xor_sync(0xffffffffu, kmin, off));
        kmax = max(kmax, (uint64_t)__shfl_xor_sync(0xffffffffu, kmax, off));
    }
    unsigned long long tot = ntile;
#pragma unroll
    for (int off = 16; off; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    if ((threadIdx.x & 31) == 0 && m) {
        atomicAdd(ctr + 0, (unsigned long long)__popc(m));
        atomicMin(ctr + 2, (unsigned long long)kmin);
        atomicMax(ctr + 3, (unsigned long long)kmax);
        atomicAdd(ctr + 10, tot);  // C_TOTK
    }
    }
}

template <class Loader>
void launch_project(const Loader& ld, int64_t n, const CamDev& cam, int sh_degree, RenderWork* w,
                    int32_t* dbg_rect, double* dbg_depth, cudaStream_t s) {
    if (n <= 0) return;
    const size_t smem = Loader::smem_bytes(ld.src);
    static int wave = -1;  // CTAs of one wave on this device (persistent grid)
    if (wave < 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // dev: GSV_PROJ_WAVES=k caps the grid at k waves of persistent CTAs
        // (descriptors staged once per CTA).  Default 0, one CTA per 128
        // splats: equal throughput in the frame-parallel mix, but a lone
        // projection runs 62 us persistent vs 41 us (no overlap between a
        // CTA's iterations)
        const char* e = getenv("GSV_PROJ_WAVES");
        const int waves = e ? atoi(e) : 0;
        wave = waves > 0 ? sms * 6 * waves : 0;
    }
    unsigned blocks = (unsigned)((n + 127) / 128);
    if (wave > 0 && blocks > (unsigned)wave) blocks = (unsigned)wave;
#define GSV_PROJ(D)                                                                                 \
    do {                                                                                            \
        if (smem > 48 * 1024)                                                                       \
            cudaFuncSetAttribute(project_kernel<Loader, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem);                                                        \
        project_kernel<Loader, D><<<blocks, 128, smem, s>>>(ld, cam, w->dkey[0], w->didx[0], w->rec, w->rect, \
                                                            w->ctr, dbg_rect, dbg_depth);           \
    } while (0)
    static int regs = -1;  // dev tuning: GSV_PROJ_REGS (register cap: occupancy vs spills), degree 1
    if (regs < 0) {
        const char* e = getenv("GSV_PROJ_REGS");
        regs = e ? atoi(e) : 80;
    }
    if (sh_degree == 1 && (regs == 72 || regs == 64)) {
        if (regs == 72)
            project_kernel<Loader, 1, 72><<<blocks, 128, smem, s>>>(ld, cam, w->dkey[0], w->didx[0], w->rec, w->rect,
                                                                     w->ctr, dbg_rect, dbg_depth);
        else
            project_kernel<Loader, 1, 64><<<blocks, 128, smem, s>>>(ld, cam, w->dkey[0], w->didx[0], w->rec, w->rect,
                                                                     w->ctr, dbg_rect, dbg_depth);
        return;
    }
    switch (sh_degree) {
        case 0: GSV_PROJ(0); break;
        case 1: GSV_PROJ(1); break;
        case 2: GSV_PROJ(2); break;
        default: GSV_PROJ(3); break;
    }
#undef GSV_PROJ
}

void launch_project_planes(const FrameSrc& src, const CamDev& cam, RenderWork* w, cudaStream_t s,
                           int32_t* dbg_rect, double* dbg_depth) {
    init_quotient_tables();
    launch_project(PlaneLoader{src}, (int64_t)src.layer_off[src.nlayers], cam, src.sh_degree, w,
                   dbg_rect, dbg_depth, s);
}

void launch_project_soa(const SoaSrc& src, const CamDev& cam, RenderWork* w, int32_t* dbg_rect,
                        double* dbg_depth, cudaStream_t s) {
    launch_project(SoaLoader{src}, src.n, cam, src.sh_degree, w, dbg_rect, dbg_depth, s);
}

// ---------------------------------------------------------------------------
// render(list[Splat2D]) (render.py:359-379): projected splats in, rects
// recomputed from cov2d exactly as render() does, then the common record /
// depth-key layout.  Depth keys are the order-preserving u64 image of the
// fp64 depth (any sign), so the stable radix sort reproduces
// argsort(depth, kind="stable") (render.py:343).  Splats with an empty rect
// draw nothing in the reference and are dropped here.
// -0.0 sorts as +0.0 and every NaN after +inf, like numpy's argsort.
__device__ __forceinline__ uint64_t orderable_key(double d) {
    if (d == 0.0) d = 0.0;
    if (d != d) return ~0ull - 1;
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

__global__ void __launch_bounds__(128) splat2d_kernel(int64_t n, const double* __restrict__ means,
                                                      const double* __restrict__ cov,
                                                      const double* __restrict__ depth,
                                                      const double* __restrict__ colors,
                                                      const double* __restrict__ opac, CamDev cam,
                                                      uint64_t* __restrict__ dkey, uint32_t* __restrict__ didx,
                                                      SplatRec* __restrict__ rec, uint2* __restrict__ rect,
                                                      unsigned long long* __restrict__ ctr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool alive = false;
    uint64_t key = ~0ull;
    uint32_t ntile = 0;
    if (i < n) {
        const double mx = means[2 * i], my = means[2 * i + 1];
        const double A = cov[4 * i], B = cov[4 * i + 1], C = cov[4 * i + 3];
        const double hm = (A - C) / 2;
        const double lam = (A + C) / 2 + sqrt(hm * hm + B * B);
        const double radius = ceil(3.0 * sqrt(np_max(lam, 0.0)));
        const double x0 = np_max(floor(mx - radius), 0.0), x1 = np_min(floor(mx + radius) + 1, (double)cam.width);
        const double y0 = np_max(floor(my - radius), 0.0), y1 = np_min(floor(my + radius) + 1, (double)cam.height);
        alive = x0 < x1 && y0 < y1;
        if (alive) {
            key = orderable_key(depth[i]);
            const double det = A * C - cov[4 * i + 1] * cov[4 * i + 1];
            const double l2e = 1.4426950408889634;
            SplatRec r;
            r.fx0 = (float)x0;
            r.fy0 = (float)y0;
            r.fx1 = (float)x1;
            r.fy1 = (float)y1;
            r.ox = (float)(mx - x0);
            r.oy = (float)(my - y0);
            r.ca = (float)(-0.5 * l2e * (C / det));
            r.cb = (float)(-l2e * (-B / det));
            r.cc = (float)(-0.5 * l2e * (A / det));
            r.r = (float)colors[3 * i];
            r.g = (float)colors[3 * i + 1];
            r.b = (float)colors[3 * i + 2];
            r.op = (float)np_max(opac[i], 0.0);  // alpha <= 0 draws nothing (render.py:326)
            r.pad = __float_as_uint(r.op > 0.f ? log2f(r.op) : -INFINITY);
            r.rx = (uint32_t)x0 | ((uint32_t)x1 << 16);
            r.ry = (uint32_t)y0 | ((uint32_t)y1 << 16);
            rec[i] = r;
            rect[i] = make_uint2(r.rx, r.ry);
            ntile = rect_tiles(r.rx, r.ry);
        }
        dkey[i] = key;
        didx[i] = (uint32_t)i;
    }
    const unsigned m = __ballot_sync(0xffffffffu, alive);
    uint64_t kmin = alive ? key : ~0ull, kmax = alive ? key : 0ull;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        kmin = min(kmin, (uint64_t)__shfl_xor_sync(0xffffffffu, kmin, off));
        kmax = max(kmax, (uint64_t)__shfl_xor_sync(0xffffffffu, kmax, off));
    }
    unsigned long long tot = ntile;
#pragma unroll
    for (int off = 16; off; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    if ((threadIdx.x & 31) == 0 && m) {
        atomicAdd(ctr + 0, (unsigned long long)__popc(m));
        atomicMin(ctr + 2, (unsigned long long)kmin);
        atomicMax(ctr + 3, (unsigned long long)kmax);
        atomicAdd(ctr + 10, tot);  // C_TOTK
    }
}

void launch_splat2d(const Splat2DSrc& src, const CamDev& cam, RenderWork* w, cudaStream_t s) {
    if (src.n <= 0) return;
    splat2d_kernel<<<(unsigned)((src.n + 127) / 128), 128, 0, s>>>(src.n, src.means, src.cov, src.depth,
                                                                   src.colors, src.opac, cam, w->dkey[0],
                                                                   w->didx[0], w->rec, w->rect, w->ctr);
}

// ---------------------------------------------------------------------------
// reconstruct_frame fold: apply_rigid then apply_residual (motion.py:165-193)
// ---------------------------------------------------------------------------
__global__ void fold_kernel(int64_t n, int shdim, double* __restrict__ pos, double* __restrict__ rot,
                            double* __restrict__ scl, double* __restrict__ opac,
                            double* __restrict__ sh, const double* __restrict__ dt,
                            const double* __restrict__ dq, const double* __restrict__ ds,
                            const double* __restrict__ dop, const double* __restrict__ dsh,
                            int* __restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double aw = dq[4 * i], ax = dq[4 * i + 1], ay = dq[4 * i + 2], az = dq[4 * i + 3];
    double* q = rot + 4 * i;
    const double bw = q[0], bx = q[1], by = q[2], bz = q[3];
    const double w = ((aw * bw - ax * bx) - ay * by) - az * bz;
    const double x = ((aw * bx + ax * bw) + ay * bz) - az * by;
    const double y = ((aw * by - ax * bz) + ay * bw) + az * bx;
    const double z = ((aw * bz + ax * by) - ay * bx) + az * bw;
    const double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
    if (nrm == 0.0) *bad = 1;
    q[0] = w / nrm;
    q[1] = x / nrm;
    q[2] = y / nrm;
    q[3] = z / nrm;
    for (int k = 0; k < 3; k++) pos[3 * i + k] = pos[3 * i + k] + dt[3 * i + k];
    for (int k = 0; k < 3; k++) scl[3 * i + k] = np_max(scl[3 * i + k] + ds[3 * i + k], 1e-7);
    opac[i] = np_min(np_max(opac[i] + dop[i], 0.0), 1.0);
    for (int k = 0; k < shdim; k++) sh[(int64_t)shdim * i + k] = sh[(int64_t)shdim * i + k] + dsh[(int64_t)shdim * i + k];
}

// All deltas of a reconstruct_frame in one pass: the splat's rigid state
// (position, rotation, scales, opacity: 11 fp64) stays in registers across
// the deltas and is read and written once; the SH coefficients are folded
// 12 at a time (their update is a plain running sum, same order).  HBM
// traffic per splat: 2 x 184 B of state + 184 B per delta, instead of
// 3 x 184 B per delta with one launch per delta.
__global__ void __launch_bounds__(256) fold_all_kernel(int64_t n, int shdim, double* __restrict__ pos,
                                                       double* __restrict__ rot, double* __restrict__ scl,
                                                       double* __restrict__ opac, double* __restrict__ sh,
                                                       const FoldTab* __restrict__ tab, int nd,
                                                       int* __restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p0 = pos[3 * i], p1 = pos[3 * i + 1], p2 = pos[3 * i + 2];
    double bw = rot[4 * i], bx = rot[4 * i + 1], by = rot[4 * i + 2], bz = rot[4 * i + 3];
    double s0 = scl[3 * i], s1 = scl[3 * i + 1], s2 = scl[3 * i + 2];
    double o = opac[i];
    bool zero = false;
    for (int d = 0; d < nd; d++) {
        const FoldTab t = tab[d];
        const double aw = __ldg(t.dq + 4 * i), ax = __ldg(t.dq + 4 * i + 1), ay = __ldg(t.dq + 4 * i + 2),
                     az = __ldg(t.dq + 4 * i + 3);
        const double w = ((aw * bw - ax * bx) - ay * by) - az * bz;
        const double x = ((aw * bx + ax * bw) + ay * bz) - az * by;
        const double y = ((aw * by - ax * bz) + ay * bw) + az * bx;
        const double z = ((aw * bz + ax * by) - ay * bx) + az * bw;
        const double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
        zero |= nrm == 0.0;
        bw = w / nrm;
        bx = x / nrm;
        by = y / nrm;
        bz = z / nrm;
        p0 = p0 + __ldg(t.dt + 3 * i);
        p1 = p1 + __ldg(t.dt + 3 * i + 1);
        p2 = p2 + __ldg(t.dt + 3 * i + 2);
        s0 = np_max(s0 + __ldg(t.ds + 3 * i), 1e-7);
        s1 = np_max(s1 + __ldg(t.ds + 3 * i + 1), 1e-7);
        s2 = np_max(s2 + __ldg(t.ds + 3 * i + 2), 1e-7);
        o = np_min(np_max(o + __ldg(t.dop + i), 0.0), 1.0);
    }
    if (zero) *bad = 1;
    pos[3 * i] = p0;
    pos[3 * i + 1] = p1;
    pos[3 * i + 2] = p2;
    rot[4 * i] = bw;
    rot[4 * i + 1] = bx;
    rot[4 * i + 2] = by;
    rot[4 * i + 3] = bz;
    scl[3 * i] = s0;
    scl[3 * i + 1] = s1;
    scl[3 * i + 2] = s2;
    opac[i] = o;
    double* shi = sh + (int64_t)shdim * i;
    for (int k0 = 0; k0 < shdim; k0 += 12) {
        double acc[12];
#pragma unroll
        for (int k = 0; k < 12; k++) acc[k] = k0 + k < shdim ? shi[k0 + k] : 0.0;
        for (int d = 0; d < nd; d++) {
            const double* dsh = tab[d].dsh + (int64_t)shdim * i + k0;
#pragma unroll
            for (int k = 0; k < 12; k++)
                if (k0 + k < shdim) acc[k] = acc[k] + __ldg(dsh + k);
        }
#pragma unroll
        for (int k = 0; k < 12; k++)
            if (k0 + k < shdim) shi[k0 + k] = acc[k];
    }
}

void launch_fold_all(int64_t n, int shdim, double* pos, double* rot, double* scl, double* opac, double* sh,
                     const FoldTab* tab, int nd, int* bad, cudaStream_t s) {
    if (n <= 0 || nd <= 0) return;
    fold_all_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, shdim, pos, rot, scl, opac, sh, tab, nd, bad);
}

void launch_fold(int64_t n, int shdim, double* pos, double* rot, double* scl, double* opac,
                 double* sh, const double* dt, const double* dq, const double* ds,
                 const double* dop, const double* dsh, int* bad, cudaStream_t s) {
    if (n <= 0) return;
    fold_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, shdim, pos, rot, scl, opac, sh, dt, dq,
                                                            ds, dop, dsh, bad);
}

}  // namespace gsv
