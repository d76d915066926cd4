// Store-bandwidth ceiling on this B200: how fast can a kernel that only
// streams float32 stores (no compute) write 16 GB? Compares 128-bit and
// 256-bit streaming stores and cudaMemsetAsync. Used to calibrate the
// roofline headroom of the env step's observation write.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st128(float4 *p, size_t n4) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    float4 v = make_float4(1.f, 0.f, 1.f, 0.f);
    for (; i < n4; i += s) __stcs(p + i, v);
}
__global__ void st256(float *p, size_t n8) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    float a = 1.f, b = 0.f;
    for (; i < n8; i += s)
        asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p + 8 * i), "f"(a), "f"(b)
                     : "memory");
}

int main() {
    size_t bytes = 16ull << 30;
    float *p;
    cudaMalloc(&p, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int kind = 0; kind < 3; kind++) {
        for (int blocks : {148 * 8, 148 * 16, 148 * 64}) {
            float best = 1e9;
            for (int it = 0; it < 5; it++) {
                cudaEventRecord(a);
                if (kind == 0) st128<<<blocks, 256>>>((float4 *)p, bytes / 16);
                else if (kind == 1) st256<<<blocks, 256>>>(p, bytes / 32);
                else cudaMemsetAsync(p, 0, bytes);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%s blocks=%d: %.3f ms  %.1f GB/s\n", kind == 0 ? "st.v4.cs" : kind == 1 ? "st.v8.cs" : "memset",
                   blocks, best, bytes / best / 1e6);
            if (kind == 2) break;
        }
    }
    return 0;
}
