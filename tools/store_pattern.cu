// Store-only replicas of the c5 step kernel's observation write pattern, to
// separate "access pattern" from "step logic" in the kernel's HBM gap.
// Every variant writes 2^20 env outputs of 15,376 B (16.1 GB) with 256-bit
// streaming stores and no compute:
//   region  : 2-warp blocks, each warp owns 32 consecutive envs (one
//             contiguous 492 KB region) and sweeps it in 1 KB warp chunks,
//             2 stores in flight per lane -- the step kernel's writer;
//             occupancy set by dynamic shared memory (like the step kernel).
//   gstride : grid-stride over the whole buffer (tools/store_ceiling.cu).
#include <cstdio>
#include <cuda_runtime.h>

static constexpr long long ENVS = 1 << 20;
static constexpr long long ENV_BYTES = 15376;
static constexpr long long ENV_F = ENV_BYTES / 4;  // 3844 floats

__device__ __forceinline__ void st8(float *p, float a, float b) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// each warp: 32 envs, contiguous; REP = stores in flight per lane
template <int REP>
__global__ void region(float *out, int envs_per_warp) {
    extern __shared__ char smem[];
    if (threadIdx.x == 1 << 30) smem[0] = 0;
    int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long e0 = warp * envs_per_warp;
    if (e0 >= ENVS) return;
    long long n8 = envs_per_warp * ENV_F / 8;  // 32-byte units in the region
    float *base = out + e0 * ENV_F;
    for (long long u = lane; u < n8; u += 32 * REP) {
#pragma unroll
        for (int r = 0; r < REP; r++) {
            long long v = u + 32 * r;
            if (v < n8) st8(base + 8 * v, 1.f, 0.f);
        }
    }
}

__global__ void gstride(float *p, long long n8) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x, s = (long long)gridDim.x * blockDim.x;
    for (; i < n8; i += s) st8(p + 8 * i, 1.f, 0.f);
}

int main() {
    size_t bytes = ENVS * ENV_BYTES;
    float *p;
    cudaMalloc(&p, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(region<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(region<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto time = [&](auto launch, const char *name) {
        float best = 1e9;
        for (int it = 0; it < 5; it++) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-48s %.3f ms  %.1f GB/s  (%.1f M env-steps/s)\n", name, best, bytes / best / 1e6,
               ENVS / best / 1e3);
    };
    // blocks per SM from dynamic smem: 31.5 KB -> 7, 27.5 KB -> 8, 14 KB -> 16
    for (int smem_kb : {32, 28, 14, 0}) {
        for (int epw : {32, 16}) {
            int threads = 64;
            long long warps = ENVS / epw;
            int blocks = (int)(warps * 32 / threads);
            char name[96];
            snprintf(name, sizeof name, "region REP=2 epw=%d smem=%dKB", epw, smem_kb);
            time([&] { region<2><<<blocks, threads, smem_kb * 1024>>>(p, epw); }, name);
            snprintf(name, sizeof name, "region REP=4 epw=%d smem=%dKB", epw, smem_kb);
            time([&] { region<4><<<blocks, threads, smem_kb * 1024>>>(p, epw); }, name);
        }
    }
    for (int blocks : {148 * 8, 148 * 64})
        time([&] { gstride<<<blocks, 256>>>(p, (long long)(bytes / 32)); }, blocks == 148 * 8 ? "gstride 1184x256" : "gstride 9472x256");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
