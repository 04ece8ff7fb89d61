// Dev microbenchmark: per-SM-sub-partition throughput of the instruction
// mixes the compositor issues (FFMA, FFMA2, FMUL2, MUFU.EX2, FSEL/FSETP).
// Each thread runs 8 independent chains; 32 warps per SM; reports warp
// instructions per cycle per SMSP for each mix (clock64 around the loop).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>

struct f2 { float x, y; };
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm volatile("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
                 "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                 : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float ex2(float x) {
    float e;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
    return e;
}
__device__ __forceinline__ float ffma(float a, float b, float c) {
    float d;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float fsel(float t, float a) {
    float r;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, 0f38D1B717;\n\tselp.f32 %0, %1, 0f00000000, p;\n\t}" : "=f"(r) : "f"(t), "f"(a));
    return r;
}

template <int MODE>
__global__ void bench(float* out, long long* cyc, int iters, float s) {
    float a[8];
    f2 p[8];
    for (int i = 0; i < 8; i++) {
        a[i] = threadIdx.x * 1e-3f + i;
        p[i] = f2{a[i], a[i] + 0.5f};
    }
    const f2 m{s, s * 0.5f}, c{0.25f, 0.125f};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) a[i] = ffma(a[i], s, a[(i + 1) & 7]);           // FFMA 3-reg
            if (MODE == 1) p[i] = fma2(p[i], m, p[(i + 1) & 7]);           // FFMA2
            if (MODE == 2) a[i] = ex2(a[i]);                               // MUFU.EX2
            if (MODE == 3) a[i] = fsel(a[i], s);                           // FSETP + FSEL
            if (MODE == 4) {                                               // compositor pair mix
                f2 q = fma2(fma2(m, p[i], c), p[i], m);
                f2 e{ex2(q.x), ex2(q.y)};
                f2 te{fsel(p[i].x, s), fsel(p[i].y, s)};
                f2 w = fma2(te, e, f2{0.f, 0.f});
                p[i] = fma2(w, m, p[i]);
                p[(i + 1) & 7] = fma2(w, c, p[(i + 1) & 7]);
            }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
    for (int i = 0; i < 8; i++) acc += a[i] + p[i].x + p[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int per_iter_instr) {
    float* out;
    long long* cyc;
    const int blocks = 148, threads = 1024, iters = 4096;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    bench<MODE><<<blocks, threads>>>(out, cyc, 16, 1.0001f);
    bench<MODE><<<blocks, threads>>>(out, cyc, iters, 1.0001f);
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < blocks; i++) c += h[i];
    c /= blocks;
    // warp instructions per SMSP: 32 warps per SM / 4 SMSPs = 8 warps each
    const double winstr = 8.0 * iters * per_iter_instr;
    printf("%-28s %7.3f warp-instr/clk/SMSP  (%.2f cycles per warp-instr)\n", name, winstr / c, c / winstr);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("FFMA (3 reg)", 8);
    run<1>("FFMA2 (3 reg pairs)", 8);
    run<2>("MUFU.EX2", 8);
    run<3>("FSETP+FSEL", 16);
    run<4>("pair mix (16 instr)", 8 * 16);
    return 0;
}
