// mma_rate2.cu -- issue cost of tcgen05.mma.cta_group::2 (M = 256 over a CTA
// pair) vs cta_group::1 (M = 128) for the trunk's small N (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_12525_b200/csrc tools/mma_rate2.cu -o tools/mma_rate2
// Clusters of 2 CTAs, one per SM; the leader's thread 0 issues R back-to-back
// bf16 MMAs (K = 16) into one accumulator and commits once (multicast to both
// CTAs' barriers). Operands are zero: only timing matters.
#include <cstdio>
#include <cuda_runtime.h>

#include "trunk_kernel.cuh"

using namespace lg;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate2_kernel(int R, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t s0 = tc::su32(sm);
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        tc::mbar_init(tc::su32(&bar), 1);
        tc::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc::tc_before();
    __syncthreads();
    cluster_sync_all();
    tc::tc_after();
    const uint32_t tmem = slot;
    const uint32_t rank = cta_rank();
    if (threadIdx.x == 0 && rank == 0) {
        constexpr uint32_t ID = tc::idesc_bf16(256, N);
        const uint64_t bd = tc::sdesc(s0 + 16384, (N / 16) * 128, 128);  // this CTA's N/2 rows of B
        const uint64_t ad = tc::sdesc(s0, 2048, 128);
        long long t0 = clock64();
        for (int i = 0; i < R; i++)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(ID), "r"(i > 0 ? 1 : 0)
                : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                tc::su32(&bar)),
            "h"((unsigned short)3)
            : "memory");
        tc::mbar_wait(tc::su32(&bar), 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if (threadIdx.x == 0) {
        tc::mbar_wait(tc::su32(&bar), 0);  // the peer's commit arrives here too
    }
    tc::tc_before();
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x < 32) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int N>
__global__ void __launch_bounds__(128, 1) rate1_kernel(int R, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t s0 = tc::su32(sm);
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        tc::mbar_init(tc::su32(&bar), 1);
        tc::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc::tc_before();
    __syncthreads();
    tc::tc_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint64_t bd = tc::sdesc(s0 + 16384, (N / 8) * 128, 128);
        const uint64_t ad = tc::sdesc(s0, 2048, 128);
        long long t0 = clock64();
        for (int i = 0; i < R; i++) tc::mma_bf16(tmem, ad, bd, tc::idesc_bf16(128, N), i > 0 ? 1u : 0u);
        tc::mma_commit(tc::su32(&bar));
        tc::mbar_wait(tc::su32(&bar), 0);
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    }
    tc::tc_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int N>
void run(long long *d) {
    const int R = 4096;
    long long c1 = 0, c2 = 0;
    cudaFuncSetAttribute(rate1_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaFuncSetAttribute(rate2_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int rep = 0; rep < 2; rep++) rate1_kernel<N><<<148, 128, 32768>>>(R, d);
    cudaMemcpy(&c1, d, 8, cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 2; rep++) rate2_kernel<N><<<148, 128, 32768>>>(R, d);
    cudaMemcpy(&c2, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("N=%3d: cta_group::1 M=128 %.1f cycles/MMA | cta_group::2 M=256 %.1f cycles/MMA  %s\n", N,
           (double)c1 / R, (double)c2 / R, cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    run<32>(d);
    run<64>(d);
    run<96>(d);
    run<128>(d);
    return 0;
}
