// racecheck_commit_repro.cu -- does compute-sanitizer racecheck model tcgen05.commit as synchronisation?
//
// The backward's racecheck reports (profiles/r01_sanitizers.md) are shared-memory write -> read pairs
// between warps that are ordered ONLY through the tensor core: warp A stores x and arrives on mbarrier
// FULL; the MMA warp waits FULL, issues a tcgen05.mma and tcgen05.commit's it to mbarrier DONE; warp B
// waits DONE and reads x.  The commit's arrive happens when the MMA completes, i.e. after FULL, so B's
// read is ordered after A's write.  This bench runs exactly that chain twice:
//   mode 0: the MMA warp signals DONE with tcgen05.commit (the kernels' pattern)
//   mode 1: the MMA warp signals DONE with a plain mbarrier.arrive after the same wait
// and checks the value B reads.  Under `compute-sanitizer --tool racecheck`, a hazard reported for mode 0
// but not for mode 1 means racecheck does not treat tcgen05.commit as a release (a false positive on the
// kernels' pattern); both modes compute the correct value.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2603_22300_b200/csrc \
//        tools/racecheck_commit_repro.cu -o /tmp/rcr && compute-sanitizer --tool racecheck /tmp/rcr
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace sfa::sm100;

// modes 2 / 3: the backward's shape -- all 32 lanes of warp A store y[lane], __syncwarp, lane 0 arrives;
// all 32 lanes of warp B wait and then OVERWRITE y[lane] (the epilogue reusing a dead operand ring)
__global__ void __launch_bounds__(96, 1) chain(int mode, int *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t full, done;
    __shared__ int x;
    __shared__ int y[32];
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2 * 16384 / 16; i += blockDim.x)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + 16 * i), "r"(0u));
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&full), 1);
        mbar_init(smem_u32(&done), 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<128>(smem_u32(&slot));
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0 && mode < 2 && lane == 0) {  // A: store x, then FULL
        x = 42 + mode;
        mbar_arrive(smem_u32(&full));
    } else if (warp == 0 && mode >= 2) {  // A, whole warp: store y[lane], __syncwarp, lane 0 -> FULL
        y[lane] = mode;
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&full));
    } else if (warp == 1 && lane == 0) {  // MMA warp: wait FULL, one MMA, DONE
        mbar_wait(smem_u32(&full), 0);
        tc_fence_after();
        umma_ss(tmem, umma_desc_sw128(base, 16, 1024), umma_desc_sw128(base + 16384, 16, 1024),
                umma_idesc_f16kind(128, 128, 0, 0, 1), 0u);
        if (mode == 0 || mode == 2) {
            umma_commit(smem_u32(&done));
        } else {
            mbar_arrive(smem_u32(&done));
        }
    } else if (warp == 2 && mode < 2 && lane == 0) {  // B: wait DONE, read x
        mbar_wait(smem_u32(&done), 0);
        out[mode] = x;
    } else if (warp == 2 && mode >= 2) {  // B, whole warp: wait DONE, overwrite y[lane]
        mbar_wait(smem_u32(&done), 0);
        y[lane] = 10 + mode;
        __syncwarp();
        if (lane == 0) out[mode] = y[31];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

int main(int argc, char **argv) {
    int *d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 34 * 1024);
    const int first = argc > 1 ? atoi(argv[1]) : 0, last = argc > 2 ? atoi(argv[2]) : 3;
    for (int mode = first; mode <= last; ++mode) chain<<<1, 96, 34 * 1024>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    int h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s: modes %d..%d, read %d %d %d %d (expect 42 43 12 13)\n", cudaGetErrorString(e), first, last, h[0], h[1],
           h[2], h[3]);
    return 0;
}
