// score_stage_bench.cu -- the two candidate SCORE stages of FlashSFA on B200, measured side by side
// (VERDICT round 1 "run the north-star design fairly").
//
// Everything else in the attention step (online softmax, P.V on tcgen05, epilogue) is the same for
// both designs, so this bench isolates what differs: producing the 256 x 128 fp32 scores of two query
// tiles against one key tile, in the form the softmax then consumes (registers of the row's thread).
//   scatter (the north star): the key tile's feature buckets (CSC_feat)
//            sit in shared memory; thread = query row, for each of its k features it walks that
//            feature's bucket and accumulates q~ * k~ into its warp's fp32 slab S_w[j][lane] (bank =
//            lane, conflict-free read-modify-write); then the row is read back (and zeroed for the
//            next tile) -- what the softmax would load.
//   tensor  (the default kernels): Q~ and K~ decompressed in shared memory (SW128 K-major), 16
//            tcgen05.mma (M128 N128 K16) per tile pair into TMEM, commit, then each row's 128 scores
//            tcgen05.ld into registers.
// Operands stay resident (no per-tile loads: the key tile's K~ (32 KB) or buckets (~(d+1)*2 + 128k*4 B)
// would arrive by TMA in both designs); codes are random, k features per row out of d = 128.
// Clocks per tile pair, one CTA per SM, 148 CTAs, max over CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_22300_b200/csrc \
//        tools/score_stage_bench.cu -o /tmp/score_stage_bench && /tmp/score_stage_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace sfa::sm100;

constexpr int D = 128, BK = 128, NTH = 256;  // 8 warps = 256 query rows

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
// k distinct features of row `row` (seeded), ascending not needed here
__device__ void row_support(uint32_t seed, int row, int k, uint8_t *f) {
    uint32_t used[4] = {0, 0, 0, 0};
    int n = 0;
    for (uint32_t c = 0; n < k; ++c) {
        const int x = (int)(hash32(seed * 7919u + (uint32_t)row * 131u + c) % D);
        if (!((used[x >> 5] >> (x & 31)) & 1u)) {
            used[x >> 5] |= 1u << (x & 31);
            f[n++] = (uint8_t)x;
        }
    }
}
__device__ __forceinline__ float val_of(uint32_t seed, int row, int u) {
    return (float)((int)(hash32(seed ^ (uint32_t)(row * 977 + u * 31)) & 255) - 128) * (1.f / 64.f);
}

// ---------------------------------------------------------------- scatter over feature buckets
template <int K>
__global__ void __launch_bounds__(NTH, 1) scatter_kernel(int tiles, unsigned long long *out, float *sink) {
    extern __shared__ __align__(16) uint8_t sm[];
    float *slab = reinterpret_cast<float *>(sm);                    // [8 warps][BK][32] fp32 = 128 KB
    uint16_t *off = reinterpret_cast<uint16_t *>(sm + 8 * BK * 32 * 4);  // [D + 1]
    uint32_t *ent = reinterpret_cast<uint32_t *>(sm + 8 * BK * 32 * 4 + 272);  // [BK * K] = j << 16 | bf16(val)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
    // key tile buckets (counting sort of the tile's BK*K (key, feature) entries by feature), built once
    if (threadIdx.x == 0) {
        uint16_t cnt[D];
        for (int f = 0; f < D; ++f) cnt[f] = 0;
        uint8_t fs[K];
        for (int j = 0; j < BK; ++j) {
            row_support(12345u + blockIdx.x, j, K, fs);
            for (int u = 0; u < K; ++u) ++cnt[fs[u]];
        }
        off[0] = 0;
        for (int f = 0; f < D; ++f) off[f + 1] = (uint16_t)(off[f] + cnt[f]);
        for (int f = 0; f < D; ++f) cnt[f] = off[f];
        for (int j = 0; j < BK; ++j) {
            row_support(12345u + blockIdx.x, j, K, fs);
            for (int u = 0; u < K; ++u) {
                const float kv = val_of(999u, j, u);
                ent[cnt[fs[u]]++] = ((uint32_t)j << 16) | (__float_as_uint(kv) >> 16);
            }
        }
    }
    float *myslab = slab + warp * BK * 32;
    for (int j = 0; j < BK; ++j) myslab[j * 32 + lane] = 0.f;
    uint8_t qf[K];
    float qv[K];
    row_support(777u + blockIdx.x, r, K, qf);
    for (int u = 0; u < K; ++u) qv[u] = val_of(555u, r, u);
    __syncthreads();
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < tiles; ++it) {
        // scatter: E[|bucket|] = BK * K / D entries per feature
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int f = qf[u];
            const int e0 = off[f], e1 = off[f + 1];
            for (int e = e0; e < e1; ++e) {
                const uint32_t x = ent[e];
                float *dst = myslab + (x >> 16) * 32 + lane;
                *dst = fmaf(qv[u], __uint_as_float(x << 16), *dst);
            }
        }
        __syncwarp();
        // the softmax's read of the row (and the zeroing for the next key tile)
#pragma unroll 8
        for (int j = 0; j < BK; ++j) {
            acc += myslab[j * 32 + lane];
            myslab[j * 32 + lane] = 0.f;
        }
        __syncwarp();
    }
    long long t1 = clock64();
    if (acc == 1234.5f) sink[0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
}

// ---------------------------------------------------------------- tcgen05 on decompressed tiles
template <int K>
__global__ void __launch_bounds__(NTH + 32, 1) tensor_kernel(int tiles, unsigned long long *out, float *sink) {
    extern __shared__ __align__(16) uint8_t sm[];  // base rounded up to 1024 below
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    const uint32_t qa = base, ka = base + 2 * 32768;  // Q~ two tiles (64 KB), K~ one tile (32 KB)
    for (int i = threadIdx.x; i < 3 * 32768 / 16; i += blockDim.x)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0u));
    __syncthreads();
    if (threadIdx.x < NTH) {  // decompress: thread r writes Q~ row r (of 256) and K~ row r (< 128)
        const int r = threadIdx.x;
        uint8_t f[K];
        row_support(777u + blockIdx.x, r, K, f);
        const uint32_t tile = qa + (r >> 7) * 32768;
        const int rr = r & 127;
        for (int u = 0; u < K; ++u) {
            const float v = val_of(555u, r, u);
            const uint32_t adr = tile + (f[u] >> 6) * 128 * 128 + rr * 128 + ((((f[u] >> 3) & 7) ^ (rr & 7)) << 4) + (f[u] & 7) * 2;
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(adr), "h"((uint16_t)(__float_as_uint(v) >> 16)));
        }
        if (r < BK) {
            row_support(12345u + blockIdx.x, r, K, f);
            for (int u = 0; u < K; ++u) {
                const float v = val_of(999u, r, u);
                const uint32_t adr = ka + (f[u] >> 6) * 128 * 128 + r * 128 + ((((f[u] >> 3) & 7) ^ (r & 7)) << 4) + (f[u] & 7) * 2;
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(adr), "h"((uint16_t)(__float_as_uint(v) >> 16)));
            }
        }
    }
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (threadIdx.x >= NTH) tmem_alloc<256>(smem_u32(&slot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x >> 5;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < tiles; ++it) {
        if (threadIdx.x == NTH) {  // issuer: S_t = Q~_t K~^T for both tiles
            tc_fence_after();
            for (int kk = 0; kk < D / 16; ++kk)
                for (int t = 0; t < 2; ++t)
                    umma_ss(tmem + t * 128, umma_desc_sw128(qa + t * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                            umma_desc_sw128(ka + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                            umma_idesc_f16kind(128, 128, 0, 0, 1), kk > 0);
            umma_commit(smem_u32(&bar));
        }
        if (threadIdx.x < NTH) {  // the softmax's read of its row
            mbar_wait(smem_u32(&bar), it & 1);
            tc_fence_after();
            const uint32_t ts = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
            uint32_t s[4][32];
            tmem_ld32(ts, s[0]);
            tmem_ld32(ts + 32, s[1]);
            tmem_ld32(ts + 64, s[2]);
            tmem_ld32(ts + 96, s[3]);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 32; ++c) acc += __uint_as_float(s[q][c]);
            tc_fence_before();
        }
        __syncthreads();  // S may be overwritten by the next tile's MMAs
    }
    long long t1 = clock64();
    if (acc == 1234.5f) sink[0] = acc;
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x >= NTH) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <typename Kern>
double run(Kern k, int threads, size_t smem, int tiles) {
    unsigned long long *d;
    float *sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, threads, smem>>>(tiles, d, sink);
    k<<<148, threads, smem>>>(tiles, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return -1;
    }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    cudaFree(d);
    cudaFree(sink);
    return (double)mx / tiles;
}

int main() {
    const int tiles = 256;
    const size_t s_sc = 8 * BK * 32 * 4 + 272 + BK * 128 * 4;
    printf("score stage for a 256-query x 128-key tile pair (32,768 pairs), d = 128, one CTA per SM, clk per tile pair\n");
    printf("(the MUFU floor of the same pairs is 2,048 clk: 16 ex2/clk/SM; tensor floor of S alone 1,024 clk)\n");
    double t;
    t = run(scatter_kernel<4>, NTH, s_sc, tiles);   printf("scatter over feature buckets  k =  4: %8.0f clk\n", t);
    t = run(scatter_kernel<8>, NTH, s_sc, tiles);   printf("scatter over feature buckets  k =  8: %8.0f clk\n", t);
    t = run(scatter_kernel<16>, NTH, s_sc, tiles);  printf("scatter over feature buckets  k = 16: %8.0f clk\n", t);
    t = run(scatter_kernel<32>, NTH, s_sc, tiles);  printf("scatter over feature buckets  k = 32: %8.0f clk\n", t);
    const size_t s_tc = 3 * 32768 + 1024;
    t = run(tensor_kernel<4>, NTH + 32, s_tc, tiles);  printf("tcgen05 on decompressed tiles k =  4: %8.0f clk\n", t);
    t = run(tensor_kernel<16>, NTH + 32, s_tc, tiles); printf("tcgen05 on decompressed tiles k = 16: %8.0f clk\n", t);
    return 0;
}
