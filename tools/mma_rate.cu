// mma_rate.cu -- tcgen05.mma issue rate for the policy trunk's shapes (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_12525_b200/csrc tools/mma_rate.cu -o tools/mma_rate
// One CTA per SM; one thread issues R back-to-back bf16 MMAs (M = 128, K = 16,
// N in {32, 64, 128, 256}) into one TMEM accumulator, A from shared memory (SS)
// or TMEM (TS), then commits once. Prints cycles per MMA and the implied
// per-SM MAC rate. Operands are zero (only timing matters).
#include <cstdio>
#include <cuda_runtime.h>

#include "trunk_kernel.cuh"

using namespace lg;

template <int N, bool TS, int NACC = 1, int CEVERY = 0>
__global__ void __launch_bounds__(128, 1) rate_kernel(int R, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const uint32_t s0 = tc::su32(sm);
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        tc::mbar_init(tc::su32(&bar), 1);
        tc::mbar_init(tc::su32(&bar2), (1 << 20) - 1);
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
        constexpr uint32_t ID = tc::idesc_bf16(128, N);
        const uint64_t bd = tc::sdesc(s0 + 16384, (N / 8) * 128, 128);
        const uint64_t ad = tc::sdesc(s0, 2048, 128);
        if (TS) tc::tmem_cp_128x256b(tmem + 256, ad);
        long long t0 = clock64();
        for (int i = 0; i < R; i++) {
            const uint32_t d = tmem + (uint32_t)((i % NACC) * (N < 64 ? N : 64));
            if (TS) tc::mma_bf16_ts(d, tmem + 256, bd, ID, i >= NACC);
            else tc::mma_bf16(d, ad, bd, ID, i >= NACC);
            if (CEVERY && (i + 1) % CEVERY == 0) tc::mma_commit(tc::su32(&bar2));
        }
        tc::mma_commit(tc::su32(&bar));
        tc::mbar_wait(tc::su32(&bar), 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc::tc_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// the trunk's conv2 pattern: A walks 36 shared 4 KB blocks, B three 3 KB
// blocks, D seven 32-column pixels; VARN: N (and so the idesc) varies at run time
template <bool VARN>
__global__ void __launch_bounds__(128, 1) pattern_kernel(int R, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t s0 = tc::su32(sm);
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
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
        const uint64_t da = tc::sdesc(s0, 2048, 128), db = tc::sdesc(s0 + 147456, 1536, 128);
        long long t0 = clock64();
        for (int i = 0; i < R; i++) {
            const int c = i % 9;
            const int n = VARN ? (c == 0 || c == 8 ? 32 : c == 1 || c == 7 ? 64 : 96) : 96;
            tc::mma_bf16(tmem + 32u * (i % 5), da + (((uint32_t)(i % 36) * 4096u) >> 4),
                         db + (((uint32_t)(i % 3) * 3072u) >> 4), tc::idesc_bf16(128, n), 1u);
        }
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

// the trunk's conv2 rows exactly: 27 MMAs per row (3 dy x 9 blocks, N = 32/64/96
// at the edges, D ranges overlapping), the conv1 ring cycling over 4 rows
__global__ void __launch_bounds__(128, 1) conv2_rows_kernel(int rows, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t s0 = tc::su32(sm);
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
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
    if (threadIdx.x < 32) {
        const uint64_t d_ring = tc::sdesc(s0, 2048, 128), d_w2 = tc::sdesc(s0 + 147456, 1536, 128);
        long long t0 = clock64();
        for (int y = 0; y < rows; y++) {
            const uint32_t acc = tmem + (uint32_t)(y & 1) * 224u;
            uint64_t dr[3];
            for (int dy = 0; dy < 3; dy++) dr[dy] = d_ring + ((uint32_t)(((y + dy) & 3) * 9) * 4096u >> 4);
            if (tc::elect_one()) {
#pragma unroll
                for (int dy = 0; dy < 3; dy++)
#pragma unroll
                    for (int c = 0; c < 9; c++) {
                        const int xlo = c - 2 > 0 ? c - 2 : 0, xhi = c < 6 ? c : 6;
                        const int jb = xlo - c + 2, n = 32 * (xhi - xlo + 1);
                        tc::mma_bf16(acc + 32u * xlo, dr[dy] + ((uint32_t)c * 4096u >> 4),
                                     d_w2 + ((uint32_t)(dy * 3072 + jb * 512) >> 4), tc::idesc_bf16(128, n), 1u);
                    }
            }
            __syncwarp();
        }
        if (tc::elect_one()) tc::mma_commit(tc::su32(&bar));
        __syncwarp();
        tc::mbar_wait(tc::su32(&bar), 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
    }
    tc::tc_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

void run_conv2_rows(long long *d) {
    const int rows = 200;
    cudaFuncSetAttribute(conv2_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    conv2_rows_kernel<<<148, 128, 200 * 1024>>>(rows, d);
    conv2_rows_kernel<<<148, 128, 200 * 1024>>>(rows, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("conv2 rows: %.1f cycles/row, %.1f cycles/MMA %s\n", (double)c / rows, (double)c / rows / 27,
           cudaGetErrorString(cudaGetLastError()));
}

template <bool VARN>
void run_pattern(long long *d) {
    const int R = 4096;
    cudaFuncSetAttribute(pattern_kernel<VARN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    pattern_kernel<VARN><<<148, 128, 160 * 1024>>>(R, d);
    pattern_kernel<VARN><<<148, 128, 160 * 1024>>>(R, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("pattern varN=%d: %.1f cycles/MMA %s\n", (int)VARN, (double)c / R, cudaGetErrorString(cudaGetLastError()));
}

template <int N, bool TS, int NACC = 1, int CEVERY = 0>
void run(long long *d) {
    const int R = 4096;
    cudaFuncSetAttribute(rate_kernel<N, TS, NACC, CEVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    rate_kernel<N, TS, NACC, CEVERY><<<148, 128, 32768>>>(R, d);
    rate_kernel<N, TS, NACC, CEVERY><<<148, 128, 32768>>>(R, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("%s N=%3d acc=%d commit/%d: %.1f cycles/MMA, %.0f MAC/cycle/SM %s\n", TS ? "TS" : "SS", N, NACC, CEVERY, (double)c / R,
           128.0 * N * 16 * R / c, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8);
    run<96, false>(d);
    run_pattern<false>(d);
    run_pattern<true>(d);
    run_conv2_rows(d);
    return 0;
}
