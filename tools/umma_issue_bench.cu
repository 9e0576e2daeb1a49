// umma_issue_bench.cu -- does the way tcgen05.mma is ISSUED limit its throughput?
//
// tools/umma_bench.cu measured ~85 clk per M=128 instruction for N = 64 and N = 128 alike (the tensor
// floor is N/2 clk: 32 / 64), and 128 clk for N = 256.  A per-instruction issue cost of ~85 clk would
// explain all three.  The kernels issue from `if (lane == 0)` with descriptors in ordinary registers,
// which ptxas wraps in an R2UR + ELECT + BRA.U.ANY waterfall per instruction.  This bench compares
//   A: that style (one lane, descriptors computed per instruction),
//   B: the whole warp converged, descriptors warp-uniform, one lane elected inside the asm (elect.sync),
// for SS N = 64 / 128 / 256 and TS N = 128, one CTA per SM, zero operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_22300_b200/csrc \
//        tools/umma_issue_bench.cu -o /tmp/umma_issue_bench && /tmp/umma_issue_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace sfa::sm100;

__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

template <int MODE, bool ELECT>
__device__ __forceinline__ void issue8(uint32_t tmem, uint32_t A, uint32_t B, uint32_t V) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0 || MODE == 1 || MODE == 2) {  // SS, N = 128 / 64 / 256
            constexpr int N = MODE == 0 ? 128 : (MODE == 1 ? 64 : 256);
            const uint64_t ad = umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(B + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
            constexpr uint32_t id = umma_idesc_f16kind(128, N, 0, 0, 1);
            if (ELECT) umma_ss_elect(tmem, ad, bd, id, kk > 0);
            else umma_ss(tmem, ad, bd, id, kk > 0);
        } else if (MODE == 4 || MODE == 5) {  // TS S with A (Q~) in TMEM, N = 64 / 128 (B = K~, K-major)
            constexpr int N = MODE == 4 ? 64 : 128;
            const uint64_t bd = umma_desc_sw128(B + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
            constexpr uint32_t id = umma_idesc_f16kind(128, N, 0, 0, 1);
            if (ELECT) umma_ts_elect(tmem + 256, tmem + 128 + kk * 8, bd, id, kk > 0);
            else umma_ts(tmem + 256, tmem + 128 + kk * 8, bd, id, kk > 0);
        } else {  // TS P.V, N = 128
            const uint64_t bd = umma_desc_sw128(V + kk * 2048, 16384, 1024);
            constexpr uint32_t id = umma_idesc_f16kind(128, 128, 0, 1, 0);
            if (ELECT) umma_ts_elect(tmem + 256, tmem + kk * 8, bd, id, 1);
            else umma_ts(tmem + 256, tmem + kk * 8, bd, id, 1);
        }
    }
}

template <int MODE, bool ELECT>
__global__ void __launch_bounds__(128, 1) bench(int reps, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0u));
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&slot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
    const uint32_t A = base, B = base + 32768, V = base + 98304;
    if (ELECT ? threadIdx.x < 32 : threadIdx.x == 0) {
        long long t0 = 0;
        uint32_t ph = 0;
        for (int rep = -2; rep < reps; ++rep) {
            if (rep == 0) {
                if (ELECT) umma_commit_elect(smem_u32(&bar)); else umma_commit(smem_u32(&bar));
                mbar_wait(smem_u32(&bar), ph);
                ph ^= 1;
                t0 = clock64();
            }
            issue8<MODE, ELECT>(tmem, A, B, V);
        }
        if (ELECT) umma_commit_elect(smem_u32(&bar)); else umma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), ph);
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) {
            out[blockIdx.x * 2] = (unsigned long long)(t1 - t0);
            out[blockIdx.x * 2 + 1] = (unsigned long long)reps * 8;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int MODE, bool ELECT>
void run(const char *name, double floor_clk) {
    unsigned long long *d;
    cudaMalloc(&d, 148 * 2 * 8);
    auto k = bench<MODE, ELECT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
    k<<<148, 128, 170 * 1024>>>(400, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    unsigned long long h[2 * 148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = (double)h[2 * i] > mx ? (double)h[2 * i] : mx;
    const double cpm = mx / (double)h[1];
    printf("%-52s %s  %7.1f clk/MMA (floor %5.1f) -> %5.1f%%\n", name, ELECT ? "elect.sync, warp converged" :
           "one lane (if lane == 0)   ", cpm, floor_clk, 100.0 * floor_clk / cpm);
    cudaFree(d);
}

int main() {
    run<0, false>("SS M128 N128 K16 bf16", 64);
    run<0, true>("SS M128 N128 K16 bf16", 64);
    run<1, false>("SS M128 N64  K16 bf16", 32);
    run<1, true>("SS M128 N64  K16 bf16", 32);
    run<2, false>("SS M128 N256 K16 bf16", 128);
    run<2, true>("SS M128 N256 K16 bf16", 128);
    run<3, false>("TS M128 N128 K16 fp16 (P.V, A in TMEM)", 64);
    run<3, true>("TS M128 N128 K16 fp16 (P.V, A in TMEM)", 64);
    run<4, false>("TS M128 N64  K16 bf16 (S, A = Q~ in TMEM)", 32);
    run<4, true>("TS M128 N64  K16 bf16 (S, A = Q~ in TMEM)", 32);
    run<5, true>("TS M128 N128 K16 bf16 (S, A = Q~ in TMEM)", 64);
    return 0;
}
