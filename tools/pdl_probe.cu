// Programmatic-dependent-launch semantics probe (B200).
//   T1: A (long, triggers at start) -> B (PDL, no griddepcontrol.wait) -> C (plain):
//       does C see all of A's writes (stream completion order kept)?
//   T2: A -> B (PDL, no wait) -> C (PDL, griddepcontrol.wait): same question for
//       a PDL successor that waits on B only.
//   T3: A -> B (PDL, no wait) -> event: does the event include A's duration?
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void gd_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void kA(int *out, int n, unsigned long long ns) {
    trigger();
    const unsigned long long t0 = gtime();
    while (gtime() - t0 < ns) {
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = 1;
}
__global__ void kB(int *flag) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *flag = 1;
}
__global__ void kC(const int *out, int n, int *zeros, int wait) {
    if (wait) gd_wait();
    int z = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) z += out[i] == 0;
    if (z) atomicAdd(zeros, z);
}

static void launch(void (*f)(int *), int *a, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t c = {};
    c.gridDim = 1;
    c.blockDim = 32;
    c.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl;
    c.attrs = at;
    c.numAttrs = 1;
    cudaLaunchKernelEx(&c, f, a);
}
static void launchC(const int *o, int n, int *z, int wait, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t c = {};
    c.gridDim = 148;
    c.blockDim = 256;
    c.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl;
    c.attrs = at;
    c.numAttrs = 1;
    cudaLaunchKernelEx(&c, kC, o, n, z, wait);
}

int main() {
    const int n = 1 << 22;
    int *out, *flag, *zeros;
    cudaMalloc(&out, n * 4);
    cudaMalloc(&flag, 4);
    cudaMalloc(&zeros, 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int test = 1; test <= 3; test++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaMemsetAsync(out, 0, n * 4, s);
            cudaMemsetAsync(zeros, 0, 4, s);
            cudaEventRecord(e0, s);
            kA<<<148, 256, 0, s>>>(out, n, 2000000ull);  // 2 ms
            launch(kB, flag, s, true);
            if (test == 3) cudaEventRecord(e1, s);
            if (test == 1) launchC(out, n, zeros, 0, s, false);
            if (test == 2) launchC(out, n, zeros, 1, s, true);
            if (test != 3) cudaEventRecord(e1, s);
            cudaStreamSynchronize(s);
            int z = -1;
            cudaMemcpy(&z, zeros, 4, cudaMemcpyDeviceToHost);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("T%d rep %d: zeros seen by C = %d, event span %.3f ms (A = 2 ms) %s\n", test, rep,
                   test == 3 ? 0 : z, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // T4: the same chain captured in a graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaMemsetAsync(zeros, 0, 4, s);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaMemsetAsync(out, 0, n * 4, s);
    kA<<<148, 256, 0, s>>>(out, n, 2000000ull);
    launch(kB, flag, s, true);
    launchC(out, n, zeros, 1, s, true);
    cudaStreamEndCapture(s, &g);
    cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; rep++) {
        cudaMemsetAsync(zeros, 0, 4, s);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        int z = -1;
        cudaMemcpy(&z, zeros, 4, cudaMemcpyDeviceToHost);
        printf("T4 graph rep %d: zeros = %d (instantiate %s, %s)\n", rep, z, cudaGetErrorString(ie),
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
