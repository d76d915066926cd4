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
#include <cuda_fp16.h>
#include <stdint.h>

#include "env_kernels.cuh"

namespace lg {

struct Conv1Div {  // runtime divisors of the index math (mul-hi + shift)
    FastDiv oo, pw, np, g;
};

// Shared memory: T [G][9][16][RS] tap tables (bias folded into tap 0 of
// group 0), S [G][16][RS] = sum over the 9 taps (a 3x3 neighbourhood whose
// cells all carry the same channel mask -- the border around the map in an
// egocentric window -- is one lookup instead of nine), the env's channel
// mask per cell and group (bytes), and the env's bits.
template <int KC, bool BF16>
__global__ void __launch_bounds__(256) conv1_bits_kernel(const uint32_t *__restrict__ bits, long long B, int C,
                                                         int OH, int OW, const float *__restrict__ w,
                                                         const float *__restrict__ bias, int K, void *out,
                                                         int relu, int nhwc, int EB, const Conv1Div dv) {
    extern __shared__ __align__(16) float csm[];
    constexpr int KP = 4 * KC;  // padded output channels per table row
    constexpr int RS = KP + 4;  // row stride (floats): rows land 20 banks apart, not 16
    const int G = (C + 3) >> 2;
    float *T = csm;  // [G][9][16][RS]
    const int rows = G * 9 * 16;
    float *S = T + (size_t)rows * RS;  // [G][16][RS]
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
            T[(size_t)i * RS + k] = s;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * 16 * KP; i += blockDim.x) {
        const int k = i % KP, m = (i / KP) & 15, g = i / (16 * KP);
        float s = 0.0f;
        for (int tap = 0; tap < 9; tap++) s += T[((size_t)(g * 9 + tap) * 16 + m) * RS + k];
        S[((size_t)g * 16 + m) * RS + k] = s;
    }
    const int OO = OH * OW, PE = C * OO;
    // EB consecutive envs per block iteration (fewer barriers, fuller rounds)
    const int NW = (EB * PE + 31) / 32 + 1;
    uint8_t *mk = reinterpret_cast<uint8_t *>(S + (size_t)G * 16 * RS);  // [EB][G][OO]
    uint32_t *eb = reinterpret_cast<uint32_t *>(mk + (((size_t)EB * G * OO + 15) & ~(size_t)15));
    const int PH = OH - 2, PW = OW - 2, NP = PH * PW;
    const unsigned long long total_words = ((unsigned long long)B * PE + 31) / 32;
    for (long long env0 = (long long)blockIdx.x * EB; env0 < B; env0 += (long long)gridDim.x * EB) {
        const int ne = B - env0 < EB ? (int)(B - env0) : EB;
        __syncthreads();  // tables built / previous envs consumed
        const unsigned long long g0 = (unsigned long long)env0 * PE, w0 = g0 >> 5;
        const uint32_t sh = (uint32_t)(g0 & 31);
        for (int i = threadIdx.x; i < NW; i += blockDim.x) {
            const uint32_t lo = w0 + i < total_words ? bits[w0 + i] : 0u;
            const uint32_t hi = w0 + i + 1 < total_words ? bits[w0 + i + 1] : 0u;
            eb[i] = __funnelshift_r(lo, hi, sh);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < ne * G * OO; i += blockDim.x) {  // channel mask per env, group, cell
            const int eg = (int)fdiv(dv.oo, (uint32_t)i), cell = i - eg * OO, e = (int)fdiv(dv.g, (uint32_t)eg),
                      g = eg - e * G;
            int m = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int c = g * 4 + j;
                if (c < C) {
                    const int b = e * PE + c * OO + cell;
                    m |= (int)((eb[b >> 5] >> (b & 31)) & 1u) << j;
                }
            }
            mk[i] = (uint8_t)m;
        }
        __syncthreads();
        const int lg_eb = __ffs(EB) - 1;
        for (int it = threadIdx.x; it < ne * NP; it += blockDim.x) {
            int e, px;
            if (nhwc == 2) {  // envs fastest: a warp's 16-byte stores fill whole core-matrix rows
                if (ne == EB) {
                    e = it & (EB - 1);
                    px = it >> lg_eb;
                } else {
                    px = it / ne;
                    e = it - px * ne;
                }
            } else {
                e = (int)fdiv(dv.np, (uint32_t)it);
                px = it - e * NP;
            }
            const long long env = env0 + e;
            const int y = (int)fdiv(dv.pw, (uint32_t)px), x = px - y * PW;
            float4 acc[KC];
#pragma unroll
            for (int q = 0; q < KC; q++) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int g = 0; g < G; g++) {
                const uint8_t *mg = mk + (e * G + g) * OO + y * OW + x;
                int ms[9];
#pragma unroll
                for (int tap = 0; tap < 9; tap++) ms[tap] = mg[(tap / 3) * OW + tap % 3];
                bool uni = true;
#pragma unroll
                for (int tap = 1; tap < 9; tap++) uni &= ms[tap] == ms[0];
                if (uni) {
                    const float4 *row = reinterpret_cast<const float4 *>(S + ((size_t)g * 16 + ms[0]) * RS);
#pragma unroll
                    for (int q = 0; q < KC; q++) {
                        const float4 v = row[q];
                        acc[q].x += v.x;
                        acc[q].y += v.y;
                        acc[q].z += v.z;
                        acc[q].w += v.w;
                    }
                } else {
#pragma unroll
                    for (int tap = 0; tap < 9; tap++) {
                        const float4 *row =
                            reinterpret_cast<const float4 *>(T + ((size_t)(g * 9 + tap) * 16 + ms[tap]) * RS);
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
            }
            if (nhwc == 2) {  // tcgen05 tile layout (trunk_kernel.cuh): K = 16, bfloat16
                // block [env / 128][px] of 128 envs x 16 channels as UMMA K-major
                // core matrices: (k / 8, m / 8) -> 128 B of 8 rows x 8 channels
                const int m = (int)(env & 127);
                __nv_bfloat16 *blk = reinterpret_cast<__nv_bfloat16 *>(out) + ((size_t)(env >> 7) * NP + px) * 2048;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    uint32_t wd[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const float4 a4 = acc[2 * h + (j >> 1)];
                        float a = (j & 1) ? a4.z : a4.x, b = (j & 1) ? a4.w : a4.y;
                        if (relu) {
                            a = a > 0.f ? a : 0.f;
                            b = b > 0.f ? b : 0.f;
                        }
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
                        wd[j] = *reinterpret_cast<uint32_t *>(&h2);
                    }
                    *reinterpret_cast<uint4 *>(blk + ((h * 16 + (m >> 3)) * 64 + (m & 7) * 8)) =
                        make_uint4(wd[0], wd[1], wd[2], wd[3]);
                }
                continue;
            }
            if (nhwc) {  // [env][px][k]: the pixel's K channels are contiguous (vector stores)
                const size_t base = ((size_t)env * NP + px) * K;
                if (BF16 && (K & 7) == 0) {
                    uint4 *o = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(out) + base);
#pragma unroll
                    for (int q = 0; q + 1 < KC + 1; q += 2) {
                        if (4 * q >= K) break;
                        float v[8] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w, 0.f, 0.f, 0.f, 0.f};
                        if (q + 1 < KC) {
                            v[4] = acc[q + 1].x;
                            v[5] = acc[q + 1].y;
                            v[6] = acc[q + 1].z;
                            v[7] = acc[q + 1].w;
                        }
                        uint32_t wd[4];
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            float a = v[2 * j], b = v[2 * j + 1];
                            if (relu) {
                                a = a > 0.f ? a : 0.f;
                                b = b > 0.f ? b : 0.f;
                            }
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
                            wd[j] = *reinterpret_cast<uint32_t *>(&h2);
                        }
                        o[q / 2] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                    }
                } else if (!BF16 && (K & 3) == 0) {
                    float4 *o = reinterpret_cast<float4 *>(reinterpret_cast<float *>(out) + base);
#pragma unroll
                    for (int q = 0; q < KC; q++) {
                        if (4 * q >= K) break;
                        float4 v = acc[q];
                        if (relu) {
                            v.x = v.x > 0.f ? v.x : 0.f;
                            v.y = v.y > 0.f ? v.y : 0.f;
                            v.z = v.z > 0.f ? v.z : 0.f;
                            v.w = v.w > 0.f ? v.w : 0.f;
                        }
                        o[q] = v;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < KC; q++) {
                        const float a4[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int k = 4 * q + j;
                            if (k < K) {
                                float v = a4[j];
                                if (relu) v = v > 0.f ? v : 0.f;
                                if (BF16) reinterpret_cast<__nv_bfloat16 *>(out)[base + k] = __float2bfloat16_rn(v);
                                else reinterpret_cast<float *>(out)[base + k] = v;
                            }
                        }
                    }
                }
                continue;
            }
            // [env][k][px]: one base per pixel, channel planes NP apart
            const size_t base = (size_t)env * K * NP + px;
            __nv_bfloat16 *ob = reinterpret_cast<__nv_bfloat16 *>(out) + base;
            float *of = reinterpret_cast<float *>(out) + base;
#pragma unroll
            for (int q = 0; q < KC; q++) {
                const float a4[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int k = 4 * q + j;
                    if (k < K) {
                        float v = a4[j];
                        if (relu) v = v > 0.f ? v : 0.f;
                        if (BF16) ob[k * NP] = __float2bfloat16_rn(v);
                        else of[k * NP] = v;
                    }
                }
            }
        }
    }
}

// Row-triple variant for the binary observation (C = 4: the one-hot tile
// planes empty / wall / border, then the frozen plane), tile layout only (the
// lg_policy_trunk input: K = 16, bfloat16). A cell whose tile planes are
// one-hot has one of 6 codes (tile x frozen), so three cells of a row have
// one of 216 and a table per kernel row dy, indexed by the triple, holds the
// sum of that row's three taps: an output pixel is three lookups instead of
// nine. A cell that is not one-hot (never produced by the env, but the
// entry point takes any bits) marks its triples invalid, and those pixels
// sum the nine tap tables of their raw 4-bit masks instead.
struct Conv1TriDiv {
    FastDiv p;  // P = O - 2
};
__device__ __forceinline__ uint32_t onehot_code(uint32_t m) {  // 4-bit cell mask -> 0..5, or 255
    const uint32_t t = m & 7u;
    const bool ok = t != 0 && (t & (t - 1)) == 0;
    return ok ? (uint32_t)(__ffs((int)t) - 1) * 2u + (m >> 3) : 255u;
}
#ifndef LG_TRI_THREADS
#define LG_TRI_THREADS 512
#endif
#ifndef LG_TRI_EB
#define LG_TRI_EB 32  // envs per block iteration (a power of two, <= 32)
#endif
__global__ void __launch_bounds__(LG_TRI_THREADS) conv1_tri_kernel(const uint32_t *__restrict__ bits, long long B, int O,
                                                        const float *__restrict__ w,
                                                        const float *__restrict__ bias, void *out, int relu,
                                                        const Conv1TriDiv dv) {
    extern __shared__ __align__(16) float csm[];
    constexpr int C = 4, K = 16, RS = K + 4, NI = 216, EB = LG_TRI_EB;
    // Row-triple tables in half precision, 16 channels per 48-byte row (32
    // used: the rows land 12 banks apart): an output pixel reads 96 bytes of
    // shared memory, not 192 -- the kernel was bound by shared-memory
    // bandwidth. fp16 (11-bit significand) sums of three entries stay well
    // inside the bfloat16 (8-bit) rounding of the output.
    constexpr int RH = 24;            // halves per table row
    __half *TRh = reinterpret_cast<__half *>(csm);  // [3][NI][RH]
    float *T = csm + 3 * NI * RH / 2;               // [9][16][RS]: the tap tables (fallback), bias in tap 0
    for (int i = threadIdx.x; i < 3 * NI * K; i += blockDim.x) {
        const int k = i % K, idx = (i / K) % NI, dy = i / (K * NI);
        float s = dy == 0 ? bias[k] : 0.0f;
        int code = idx;
#pragma unroll
        for (int dx = 0; dx < 3; dx++) {
            const int cd = code % 6, tile = cd >> 1, frz = cd & 1;
            code /= 6;
            s += w[((k * C + tile) * 3 + dy) * 3 + dx];
            if (frz) s += w[((k * C + 3) * 3 + dy) * 3 + dx];
        }
        TRh[(dy * NI + idx) * RH + k] = __float2half_rn(s);
    }
    for (int i = threadIdx.x; i < 9 * 16 * K; i += blockDim.x) {
        const int k = i % K, m = (i / K) & 15, tap = i / (16 * K);
        float s = tap == 0 ? bias[k] : 0.0f;
#pragma unroll
        for (int c = 0; c < C; c++)
            if ((m >> c) & 1) s += w[(k * C + c) * 9 + tap];
        T[(tap * 16 + m) * RS + k] = s;
    }
    const int OO = O * O, PE = C * OO, P = O - 2, NP = P * P;
    uint8_t *tri = reinterpret_cast<uint8_t *>(T + 9 * 16 * RS);  // [EB][O][P]
    uint32_t *eb = reinterpret_cast<uint32_t *>(tri + (((size_t)EB * O * P + 15) & ~(size_t)15));
    const int NW = (EB * PE + 31) / 32 + 1;
    const unsigned long long total_words = ((unsigned long long)B * PE + 31) / 32;
    for (long long env0 = (long long)blockIdx.x * EB; env0 < B; env0 += (long long)gridDim.x * EB) {
        const int ne = B - env0 < EB ? (int)(B - env0) : EB;
        __syncthreads();  // tables built / previous envs consumed
        const unsigned long long g0 = (unsigned long long)env0 * PE, w0 = g0 >> 5;
        const uint32_t sh = (uint32_t)(g0 & 31);
        for (int i = threadIdx.x; i < NW; i += blockDim.x) {
            const uint32_t lo = w0 + i < total_words ? bits[w0 + i] : 0u;
            const uint32_t hi = w0 + i + 1 < total_words ? bits[w0 + i + 1] : 0u;
            eb[i] = __funnelshift_r(lo, hi, sh);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < ne * O; i += blockDim.x) {  // one observation row (env, y) per thread
            const int e = i / O, y = i - e * O;
            uint32_t r[C];
#pragma unroll
            for (int c = 0; c < C; c++) {
                const int b = e * PE + c * OO + y * O;  // O <= 31: the row fits one funnel shift
                r[c] = __funnelshift_r(eb[b >> 5], eb[(b >> 5) + 1], b & 31);
            }
            uint8_t *dst = tri + (size_t)i * P;
            uint32_t c0 = 0, c1 = 0;
            for (int x = 0; x < O; x++) {
                const uint32_t m = ((r[0] >> x) & 1u) | ((r[1] >> x) & 1u) << 1 | ((r[2] >> x) & 1u) << 2 |
                                   ((r[3] >> x) & 1u) << 3;
                const uint32_t c2 = onehot_code(m);
                if (x >= 2) dst[x - 2] = (uint8_t)((c0 | c1 | c2) > 5u ? 255u : c0 + 6u * c1 + 36u * c2);
                c0 = c1;
                c1 = c2;
            }
        }
        __syncthreads();
        for (int it = threadIdx.x; it < ne * NP; it += blockDim.x) {
            int e, px;
            if (ne == EB) {  // envs fastest: a warp's 16-byte stores fill whole core-matrix rows
                e = it & (EB - 1);
                px = it / EB;
            } else {
                px = it / ne;
                e = it - px * ne;
            }
            const int y = (int)fdiv(dv.p, (uint32_t)px), x = px - y * P;
            const uint8_t *t0 = tri + ((size_t)e * O + y) * P + x;
            const uint32_t i0 = t0[0], i1 = t0[P], i2 = t0[2 * P];
            float4 acc[4];
            if (max(i0, max(i1, i2)) < (uint32_t)NI) {
                const uint4 *r0 = reinterpret_cast<const uint4 *>(TRh + (0 * NI + i0) * RH);
                const uint4 *r1 = reinterpret_cast<const uint4 *>(TRh + (1 * NI + i1) * RH);
                const uint4 *r2 = reinterpret_cast<const uint4 *>(TRh + (2 * NI + i2) * RH);
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    const uint4 a = r0[q], b = r1[q], c = r2[q];
                    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w},
                                   cv[4] = {c.x, c.y, c.z, c.w};
                    float f[8];
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const __half2 h = __hadd2(__hadd2(*reinterpret_cast<const __half2 *>(&av[j]),
                                                          *reinterpret_cast<const __half2 *>(&bv[j])),
                                                  *reinterpret_cast<const __half2 *>(&cv[j]));
                        const float2 v = __half22float2(h);
                        f[2 * j] = v.x;
                        f[2 * j + 1] = v.y;
                    }
                    acc[2 * q] = make_float4(f[0], f[1], f[2], f[3]);
                    acc[2 * q + 1] = make_float4(f[4], f[5], f[6], f[7]);
                }
            } else {  // a cell that is not one-hot: the nine taps of the raw masks
#pragma unroll
                for (int q = 0; q < 4; q++) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int tap = 0; tap < 9; tap++) {
                    const int cell = (y + tap / 3) * O + x + tap % 3;
                    uint32_t m = 0;
#pragma unroll
                    for (int c = 0; c < C; c++) {
                        const int b = e * PE + c * OO + cell;
                        m |= ((eb[b >> 5] >> (b & 31)) & 1u) << c;
                    }
                    const float4 *row = reinterpret_cast<const float4 *>(T + (tap * 16 + m) * RS);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const float4 v = row[q];
                        acc[q].x += v.x;
                        acc[q].y += v.y;
                        acc[q].z += v.z;
                        acc[q].w += v.w;
                    }
                }
            }
            const long long env = env0 + e;
            const int m = (int)(env & 127);
            __nv_bfloat16 *blk = reinterpret_cast<__nv_bfloat16 *>(out) + ((size_t)(env >> 7) * NP + px) * 2048;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                uint32_t wd[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float4 a4 = acc[2 * h + (j >> 1)];
                    float a = (j & 1) ? a4.z : a4.x, b = (j & 1) ? a4.w : a4.y;
                    if (relu) {
                        a = a > 0.f ? a : 0.f;
                        b = b > 0.f ? b : 0.f;
                    }
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
                    wd[j] = *reinterpret_cast<uint32_t *>(&h2);
                }
                *reinterpret_cast<uint4 *>(blk + ((h * 16 + (m >> 3)) * 64 + (m & 7) * 8)) =
                    make_uint4(wd[0], wd[1], wd[2], wd[3]);
            }
        }
    }
}

}  // namespace lg
