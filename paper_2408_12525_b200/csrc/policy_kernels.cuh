// policy_kernels.cuh -- the policy consumer of the observation.
//
// The reference's ConvPolicy (levelgen/nets.py:150-183) starts its trunk with
// Conv2d(C, K, kernel_size=3) (valid) + ReLU over the float32 observation
// [B, C, O, O]. Every input element is 0 or 1, so a 3x3 tap over C channels
// contributes the sum of the weights of the set channels: with the channels
// split into groups of four, one tap of one group is a lookup of a 16-entry
// table of K-vectors. conv1_bits_kernel reads the packed observation stream
// (LG_OBS_BITS, 1 bit per element) instead of 32-bit floats, builds the
// tables once per CTA in shared memory (bias folded into tap 0), and writes
// relu(conv1) in float32 or bfloat16: the HBM traffic is the output plus
// 1/32 of the float32 input.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace lg {

template <int KC, bool BF16>
__global__ void __launch_bounds__(256) conv1_bits_kernel(const uint32_t *__restrict__ bits, long long B, int C,
                                                         int OH, int OW, const float *__restrict__ w,
                                                         const float *__restrict__ bias, int K, void *out,
                                                         int relu) {
    extern __shared__ __align__(16) float csm[];
    constexpr int KP = 4 * KC;  // padded output channels per table row
    const int G = (C + 3) >> 2;
    float *T = csm;  // [G][9][16][KP]
    const int rows = G * 9 * 16;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
        const int m = i & 15, tap = (i >> 4) % 9, g = i / (9 * 16);
        for (int k = 0; k < KP; k++) {
            float s = (g == 0 && tap == 0 && k < K) ? bias[k] : 0.0f;
            if (k < K) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int c = g * 4 + j;
                    if (c < C && ((m >> j) & 1)) s += w[((size_t)k * C + c) * 9 + tap];
                }
            }
            T[(size_t)i * KP + k] = s;
        }
    }
    const int OO = OH * OW, PE = C * OO;
    const int NW = (PE + 31) / 32 + 1;
    uint32_t *eb = reinterpret_cast<uint32_t *>(T + (size_t)rows * KP);
    const int PH = OH - 2, PW = OW - 2, NP = PH * PW;
    const unsigned long long total_words = ((unsigned long long)B * PE + 31) / 32;
    for (long long env = blockIdx.x; env < B; env += gridDim.x) {
        __syncthreads();  // tables built / previous env's bits consumed
        const unsigned long long g0 = (unsigned long long)env * PE, w0 = g0 >> 5;
        const uint32_t sh = (uint32_t)(g0 & 31);
        for (int i = threadIdx.x; i < NW; i += blockDim.x) {
            const uint32_t lo = w0 + i < total_words ? bits[w0 + i] : 0u;
            const uint32_t hi = w0 + i + 1 < total_words ? bits[w0 + i + 1] : 0u;
            eb[i] = __funnelshift_r(lo, hi, sh);
        }
        __syncthreads();
        for (int px = threadIdx.x; px < NP; px += blockDim.x) {
            const int y = px / PW, x = px - y * PW;
            float4 acc[KC];
#pragma unroll
            for (int q = 0; q < KC; q++) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int tap = 0; tap < 9; tap++) {
                const int cell = (y + tap / 3) * OW + x + tap % 3;
                for (int g = 0; g < G; g++) {
                    int m = 0;
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const int c = g * 4 + j;
                        if (c < C) {
                            const int b = c * OO + cell;
                            m |= (int)((eb[b >> 5] >> (b & 31)) & 1u) << j;
                        }
                    }
                    const float4 *row = reinterpret_cast<const float4 *>(T + ((size_t)(g * 9 + tap) * 16 + m) * KP);
#pragma unroll
                    for (int q = 0; q < KC; q++) {
                        const float4 v = row[q];
                        acc[q].x += v.x;
                        acc[q].y += v.y;
                        acc[q].z += v.z;
                        acc[q].w += v.w;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < KC; q++) {
                const float a4[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int k = 4 * q + j;
                    if (k < K) {
                        float v = a4[j];
                        if (relu) v = v > 0.f ? v : 0.f;
                        const size_t o = ((size_t)env * K + k) * NP + px;
                        if (BF16) reinterpret_cast<__nv_bfloat16 *>(out)[o] = __float2bfloat16_rn(v);
                        else reinterpret_cast<float *>(out)[o] = v;
                    }
                }
            }
        }
    }
}

}  // namespace lg
