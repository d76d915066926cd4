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
#include <cstdint>
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

// region stores with a per-warp prologue like the step kernel's: each lane
// loads its env's state (PRO bytes), spins ~ALU dependent ops, writes its
// smem image (SMW words), __syncwarp, then the warp expands smem bits to floats.
template <int PRO, int ALU, int SMW, bool DATA, int PF = 0, bool HOT = false>
__global__ void region_pro(float *out, const uint4 *state, int envs_per_warp) {
    extern __shared__ uint32_t sm[];
    int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long e0 = warp * envs_per_warp;
    if (e0 >= ENVS) return;
    uint32_t *img = sm + wib * 32 * 123;
    uint32_t acc = 0;
    if (PRO > 0) {
        const uint4 *st = state + ((HOT ? (e0 & 4095) : e0) + lane) * (PRO / 16);
#pragma unroll
        for (int i = 0; i < PRO / 16; i++) {
            uint4 v = st[i];
            acc ^= v.x + v.y * 3 + v.z * 5 + v.w * 7;
        }
    }
#pragma unroll 1
    for (int i = 0; i < ALU; i++) acc = acc * 1664525u + 1013904223u;
    for (int w = 0; w < SMW; w++) img[lane * 123 + w] = acc ^ (w * 0x9E3779B9u);
    __syncwarp();
    if (PF > 0) {  // L2 prefetch of the state of the env PF warps ahead (next wave)
        long long pe = e0 + (long long)PF * envs_per_warp + lane;
        if (pe < ENVS) {
            const char *a = reinterpret_cast<const char *>(state + pe * (PRO / 16));
            for (int i = 0; i < PRO; i += 64) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + i));
        }
    }
    long long n8 = envs_per_warp * ENV_F / 8;
    float *base = out + e0 * ENV_F;
    for (long long u = lane; u < n8; u += 64) {
#pragma unroll
        for (int r = 0; r < 2; r++) {
            long long v = u + 32 * r;
            if (v < n8) {
                uint32_t x = DATA ? (img[(v >> 2) % (32 * 123)] >> ((v & 3) * 8)) : 0x55u;
                float f[8];
#pragma unroll
                for (int j = 0; j < 8; j++) f[j] = ((x >> j) & 1u) ? 1.0f : 0.0f;
                asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(base + 8 * v),
                             "f"(f[0]), "f"(f[1]), "f"(f[2]), "f"(f[3]), "f"(f[4]), "f"(f[5]), "f"(f[6]),
                             "f"(f[7]));
            }
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
    uint4 *state;
    cudaMalloc(&state, ENVS * 128);
    cudaMemset(state, 1, ENVS * 128);
    {
        int threads = 64, blocks = (int)(ENVS / 32 * 32 / threads);
        size_t sm = 2 * 32 * 123 * 4;  // 31.5 KB: 7 blocks/SM like the step kernel
#define PRO_CASE(P, A, W, D, NAME) PRO_CASE_PF(P, A, W, D, 0, NAME)
#define PRO_CASE_PF(P, A, W, D, F, NAME)                                                              \
    cudaFuncSetAttribute(region_pro<P, A, W, D, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    time([&] { region_pro<P, A, W, D, F><<<blocks, threads, sm>>>(p, state, 32); }, NAME);
        PRO_CASE(0, 0, 0, false, "pro: none, const data")
        PRO_CASE(0, 0, 0, true, "pro: none, smem bits")
        PRO_CASE(0, 0, 122, true, "pro: smem image write, smem bits")
        PRO_CASE(128, 0, 122, true, "pro: 128B state load + image, smem bits")
        PRO_CASE(32, 0, 122, true, "pro: 32B state load + image")
        PRO_CASE(64, 0, 122, true, "pro: 64B state load + image")
        PRO_CASE(256, 0, 122, true, "pro: 256B state load + image")
        cudaFuncSetAttribute(region_pro<128, 0, 122, true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        time([&] { region_pro<128, 0, 122, true, 0, true><<<blocks, threads, sm>>>(p, state, 32); },
             "pro: 128B state load (L2-resident) + image");
        PRO_CASE(128, 2000, 122, true, "pro: load + 2000 ALU + image")
        PRO_CASE(128, 8000, 122, true, "pro: load + 8000 ALU + image")
        PRO_CASE(0, 8000, 122, true, "pro: 8000 ALU + image (no load)")
        for (int kb : {24, 14, 10}) {
            char name[96];
            snprintf(name, sizeof name, "pro: 64B load + 2000 ALU, const data, smem %d KB/block", kb);
            time([&] { region_pro<64, 2000, 0, false><<<blocks, threads, (size_t)kb * 1024>>>(p, state, 32); }, name);
        }
        PRO_CASE(64, 2000, 0, false, "pro: 64B load + 2000 ALU, const data, 31.5 KB")
    }
    for (int blocks : {148 * 8, 148 * 64})
        time([&] { gstride<<<blocks, 256>>>(p, (long long)(bytes / 32)); }, blocks == 148 * 8 ? "gstride 1184x256" : "gstride 9472x256");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
