// umma_bench.cu -- microbenchmark of tcgen05.mma issue-to-completion throughput for the shapes the
// FlashSFA sm100 kernel uses (one CTA per SM, one thread issues, operands are zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_22300_b200/csrc \
//        tools/umma_bench.cu -o /tmp/umma_bench && /tmp/umma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace sfa::sm100;

__global__ void __launch_bounds__(128, 1) bench(int mode, int reps, unsigned long long *out, int interf) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2;
    const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
        uint32_t v = 0;
        if (interf == 1) {  // random-ish bf16 values in [-2, 2): sign, exponent 126/127, random mantissa
            uint32_t h = (uint32_t)i * 2654435761u + 12345u;
            h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
            v = ((h & 0x807F807Fu) | 0x3F003F00u) ^ ((h >> 8) & 0x00800080u);
        }
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(v));
    }
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&bar2), 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&slot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (threadIdx.x >= 32 && interf >= 2) {  // warps 1-3 generate interference until the MMAs finish
        const int w = threadIdx.x >> 5;
        const uint32_t lane_off = (uint32_t)(w * 32) << 16;
        uint32_t r[32];
        for (int i = 0; i < 32; ++i) r[i] = i;
        while (!done) {
            if (interf == 4) {  // ALU + MUFU pressure (softmax-like): FFMA / ex2 chains
                float x = (float)threadIdx.x;
#pragma unroll 1
                for (int i = 0; i < 64; ++i) {
                    float y0 = x, y1 = x + 1.f, y2 = x + 2.f, y3 = x + 3.f;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y0));
                        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y1));
                        y2 = fmaf(y2, 0.999f, 0.001f);
                        y3 = fmaf(y3, 0.999f, 0.001f);
                    }
                    x = y0 + y1 + y2 + y3;
                }
                r[0] += __float_as_uint(x);
            } else if (interf == 2) {  // TMEM reads + writes on columns 448.. (not used by the MMAs)
                tmem_ld32(tmem + lane_off + 448, r);
                tmem_ld_wait();
                tmem_st32(tmem + lane_off + 480, r);
                tmem_st_wait();
            } else {  // shared-memory stores (16 B per lane) to a region the MMAs do not read
                for (int i = 0; i < 16; ++i)
                    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 131072 + ((threadIdx.x * 16 + i * 512) & 16383)), "r"(r[i]));
            }
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t A = base, B = base + 32768, V = base + 65536;
        int n_mma = 0;
        long long t0 = 0;
        for (int rep = -2; rep < reps; ++rep) {
            if (rep == 0) t0 = clock64();
            switch (mode) {
                case 0:  // S: SS, M128 N128, K=128 (8 K-steps), bf16
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    n_mma += 8;
                    break;
                case 1:  // S: SS, M128 N64, K=128
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 64, 0, 0, 1), kk > 0);
                    n_mma += 8;
                    break;
                case 2:  // PV: TS, M128 N128, K=128 (8 K-steps), fp16, B MN-major
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(V + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    n_mma += 8;
                    break;
                case 3:  // S as TS: A (Q~) from TMEM, M128 N128, K=128
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    n_mma += 8;
                    break;
                case 4:  // S: SS, M128 N256, K=128
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 256, 0, 0, 1), kk > 0);
                    n_mma += 8;
                    break;
                case 5:  // PV: TS, M128 N128, K=64 x2 groups
                    for (int kk = 0; kk < 4; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(V + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    n_mma += 4;
                    break;
                case 6:  // SS N128, 2 independent accumulators interleaved
                    for (int kk = 0; kk < 8; ++kk)
                        for (int c = 0; c < 2; ++c)
                            umma_ss(tmem + 128 * c, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    n_mma += 16;
                    break;
                case 7:  // SS N64, 2 chains
                case 8:  // SS N64, 4 chains
                {
                    const int nc = mode == 7 ? 2 : 4;
                    for (int kk = 0; kk < 8; ++kk)
                        for (int c = 0; c < nc; ++c)
                            umma_ss(tmem + 64 * c, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_idesc_f16kind(128, 64, 0, 0, 1), kk > 0);
                    n_mma += 8 * nc;
                    break;
                }
                case 9:  // TS PV N128, 2 chains (D = 256, 384; A = cols 0.., 128..)
                    for (int kk = 0; kk < 8; ++kk)
                        for (int c = 0; c < 2; ++c)
                            umma_ts(tmem + 256 + 128 * c, tmem + 128 * c + kk * 8,
                                    umma_desc_sw128(V + kk * 2048, 16384, 1024), umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    n_mma += 16;
                    break;
                case 10:  // SS N128 single chain, no accumulate (no RAW on C)
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), 0);
                    n_mma += 8;
                    break;
                case 11:  // mixed: PV (TS N128, D=O) interleaved with S (SS N64) for 2 tiles -> 4 chains
                    for (int kk = 0; kk < 8; ++kk) {
                        for (int c = 0; c < 2; ++c)
                            umma_ss(tmem + 64 * c, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                    umma_idesc_f16kind(128, 64, 0, 0, 1), kk > 0);
                        if (kk < 4)
                            for (int c = 0; c < 2; ++c)
                                umma_ts(tmem + 256 + 128 * c, tmem + 128 + 32 * c + kk * 8,
                                        umma_desc_sw128(V + kk * 2048, 16384, 1024), umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    }
                    n_mma += 24;
                    break;
                case 15: {  // as 12, but B (and A of S) rotate over fresh 32 KB tiles each rep (no operand reuse)
                    const uint32_t rot = (uint32_t)((rep & 3) * 32768);
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(base + ((rot + 65536) & 131071) + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    umma_commit(smem_u32(&bar2));
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem + 128, umma_desc_sw128(base + ((rot + 32768 * ((rep >> 2) & 1)) & 131071) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(base + rot + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    umma_commit(smem_u32(&bar2));
                    n_mma += 16;
                    break;
                }
                case 12:  // PV (TS, D=O) 8 K-steps + commit, then S (SS, D=S) 8 K-steps + commit
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(V + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    umma_commit(smem_u32(&bar2));
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem + 128, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    umma_commit(smem_u32(&bar2));
                    n_mma += 16;
                    break;
                case 13:  // same 16 MMAs without the intermediate commits
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + kk * 8, umma_desc_sw128(V + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem + 128, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    n_mma += 16;
                    break;
                case 14:  // as 12, but PV reads A (P) from the TMEM columns S is about to be written into
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ts(tmem + 256, tmem + 128 + kk * 8, umma_desc_sw128(V + kk * 2048, 16384, 1024),
                                umma_idesc_f16kind(128, 128, 0, 1, 0), 1);
                    umma_commit(smem_u32(&bar2));
                    for (int kk = 0; kk < 8; ++kk)
                        umma_ss(tmem + 128, umma_desc_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_desc_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
                    umma_commit(smem_u32(&bar2));
                    n_mma += 16;
                    break;
            }
            if (rep == -1) {
                umma_commit(smem_u32(&bar));
                mbar_wait(smem_u32(&bar), 0);
                t0 = clock64();
                n_mma = 0;
            }
        }
        umma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 1);
        const long long t1 = clock64();
        out[blockIdx.x * 2] = (unsigned long long)(t1 - t0);
        out[blockIdx.x * 2 + 1] = (unsigned long long)n_mma;
        done = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 148 * 2 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
    const char *names[] = {"SS M128 N128 K16 bf16 (S, 128 keys)", "SS M128 N64  K16 bf16 (S, 64 keys)",
                           "TS M128 N128 K16 fp16 (P.V)", "TS M128 N128 K16 bf16 (S with Q~ in TMEM)",
                           "SS M128 N256 K16 bf16", "TS M128 N128 K16 fp16 (P.V, 4-step groups)",
                           "SS N128, 2 accumulators interleaved", "SS N64, 2 accumulators interleaved",
                           "SS N64, 4 accumulators interleaved", "TS N128 P.V, 2 accumulators",
                           "SS N128 single chain, accumulate=0", "mixed 2xS N64 + 2xPV N128 (mean N 85)",
                           "PV(8)+commit, S(8)+commit", "PV(8), S(8), no commits", "PV(8) reading S cols+commit, S(8)+commit",
                           "as 12, operands rotating over fresh tiles"};
    const int flop_n[] = {128, 64, 128, 128, 256, 128, 128, 64, 64, 128, 128, 85, 128, 128, 128, 128};
    const char *inames[] = {"zeros", "random operands", "zeros + TMEM ld/st by 3 warps", "zeros + smem stores by 3 warps",
                            "zeros + ALU/MUFU work by 3 warps (one on the issuer's SMSP)"};
    for (int interf : {0, 1}) {
        printf("--- %s\n", inames[interf]);
        const int grid = 148;
        for (int mode : {12, 15}) {
            bench<<<grid, 128, 170 * 1024>>>(mode, 200, d, interf);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double cpm = (double)h[0] / (double)h[1];
            const double ideal = 128.0 * flop_n[mode] / 256.0;
            printf("grid %3d  %-44s %7.1f clk/MMA (model %5.1f) -> %5.1f%% of 8192 FLOP/clk\n", grid, names[mode], cpm,
                   ideal, 100.0 * ideal / cpm);
        }
    }
    return 0;
}
