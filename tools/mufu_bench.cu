// MUFU.EX2 / FMA-pipe throughput on one B200 (nvcc -gencode arch=compute_100a,code=sm_100a -O3).
// Each thread runs ILP independent chains of ITER dependent ops; clocks per SM -> ops / clk / SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void ex2_kernel(float *out, int iters, long long *clk) {
    float v[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = -1e-3f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int ILP>
__global__ void ffma2_kernel(float *out, int iters, long long *clk) {
    float v[2 * ILP];
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) v[i] = 1e-3f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("{\n\t.reg .b64 a;\n\tmov.b64 a, {%0, %1};\n\tfma.rn.f32x2 a, a, a, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
                         : "+f"(v[2 * i]), "+f"(v[2 * i + 1]));
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}


template <int ILP>
__global__ void f2fp_kernel(float *out, int iters, long long *clk) {
    float v[2 * ILP];
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) v[i] = 1e-3f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            uint32_t r;
            asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[2 * i]), "f"(v[2 * i + 1]));
            acc ^= r;
        }
    }
    long long t1 = clock64();
    if (acc == 12345u) out[0] = 1.f;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// 2 ex2 + 1 f16x2 pack per pair, the softmax's mix.  Each ex2 feeds the next iteration (x <- -ex2(x)),
// otherwise ptxas hoists the loop-invariant MUFU ops out of the loop (an earlier version of this test
// reported 254 "ex2/clk" that way).
template <int ILP>
__global__ void mix_kernel(float *out, int iters, long long *clk) {
    float v[2 * ILP];
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 2 * ILP; ++i) v[i] = -1e-3f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            float a, b;
            uint32_t r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(v[2 * i]));
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(v[2 * i + 1]));
            asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
            acc ^= r;
            v[2 * i] = -a;
            v[2 * i + 1] = -b;
        }
    }
    long long t1 = clock64();
    if (acc == 12345u) out[0] = 1.f;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// MUFU.EX2 on f16x2 (ex2.approx.f16x2): ptxas emits two MUFU.EX2.F16 per instruction on sm_100a
template <int ILP>
__global__ void ex2h2_kernel(float *out, int iters, long long *clk) {
    uint32_t v[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = 0xBC00BC00u ^ (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
            v[i] ^= 0x80008000u;  // keep the argument negative
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s ^= v[i];
    if (s == 12345u) out[0] = 1.f;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// MUFU.EX2 with a per-lane predicate: does a lane whose predicate is off cost MUFU throughput?
// (a pair with no shared feature has logit exactly 0, its weight is a per-row
// constant; at k = 4 of d = 128 about 88 % of the pairs.)  `active` lanes of 32 run the ex2.
template <int ILP>
__global__ void ex2_pred_kernel(float *out, int iters, long long *clk, int active) {
    float v[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = -1e-3f * (threadIdx.x + i);
    const uint32_t on = (threadIdx.x & 31) < active;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p ex2.approx.ftz.f32 %0, %0;\n\t}"
                         : "+f"(v[i]) : "r"(on));
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char *name, K kern, int threads, int ops_per_iter, int iters) {
    float *out;
    long long *clk;
    cudaMalloc(&out, 4);
    cudaMalloc(&clk, 148 * sizeof(long long));
    kern<<<148, threads>>>(out, iters, clk);
    kern<<<148, threads>>>(out, iters, clk);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double ops = (double)threads * ops_per_iter * iters;
    printf("%-28s threads/SM %4d: %.2f ops/clk/SM\n", name, threads, ops / mx);
    cudaFree(out);
    cudaFree(clk);
}

template <typename K>
void run_pred(const char *name, K kern, int threads, int ops_per_iter, int iters, int active) {
    float *out;
    long long *clk;
    cudaMalloc(&out, 4);
    cudaMalloc(&clk, 148 * sizeof(long long));
    kern<<<148, threads>>>(out, iters, clk, active);
    kern<<<148, threads>>>(out, iters, clk, active);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double winstr = (double)threads / 32 * ops_per_iter * iters;
    printf("%-28s threads/SM %4d, %2d of 32 lanes on: %.2f warp-instr/clk/SM (%.2f active ex2/clk/SM)\n", name, threads,
           active, winstr / mx, winstr * active / mx);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    for (int act : {32, 16, 8, 4, 1}) run_pred("predicated ex2 ILP8", ex2_pred_kernel<8>, 512, 8, 4096, act);
    for (int th : {128, 256, 512, 1024}) {
        run("ex2.approx ILP8", ex2_kernel<8>, th, 8, 4096);
        run("ex2.approx ILP32", ex2_kernel<32>, th, 32, 1024);
        run("fma.rn.f32x2 ILP8 (elems)", ffma2_kernel<8>, th, 16, 4096);
        run("cvt.rn.f16x2.f32 ILP8 (instr)", f2fp_kernel<8>, th, 8, 4096);
        run("2 ex2 + 1 cvt f16x2 (ex2/clk)", mix_kernel<8>, th, 16, 4096);
        run("ex2.approx.f16x2 ILP8 (elems)", ex2h2_kernel<8>, th, 16, 4096);
    }
    return 0;
}
