// trunk_kernel.cuh -- the rest of the policy trunk on the 5th-gen tensor cores.
//
// Reference: levelgen/nets.py:150-183 (ConvPolicy, default arch (16, 32) convs +
// one 64-wide FC) inside ppo.collect_rollout (ppo.py:101-143). After
// conv1_bits_kernel has written relu(conv1) in the tile layout below, one CTA
// runs, for 128 environments at a time:
//
//   conv2 (16 -> 32, 3x3 valid) + bias + ReLU     -- tcgen05.mma, M = 128 envs,
//                                                    N = 32, K = 9 taps x 16
//   FC (32 * P2 * P2 -> 64), accumulated pixel by  -- tcgen05.mma, M = 128,
//   pixel straight from each conv2 output pixel       N = 64, K = 32 per pixel
//   + bias + ReLU, then the policy / value heads  -- CUDA cores, fp32
//
// so neither the conv2 activations (46.7 KB per env at obs 31) nor the FC
// input ever reach HBM. Accumulators live in TMEM (a 4-slot ring of 32-column
// conv2 pixels + the 64-column FC accumulator); operands are UMMA K-major
// core-matrix layouts (8 rows x 16 B, no swizzle) in shared memory.
//
// Data layout (all bf16, prepared by conv1_bits_kernel / the host):
//   c1  [ceil(B/128)][P1*P1][2048]: per pixel, 128 envs x 16 channels,
//       element (m, k) at ((k/8)*16 + m/8)*64 + (m%8)*8 + k%8
//   w2  [3 dy][1536]: N = 96 (taps dx = 2, 1, 0 x 32 out channels) x K = 16 in,
//       element (n, k) at ((k/8)*12 + n/8)*64 + (n%8)*8 + k%8
//   w3  [P2*P2][2048]: per conv2 pixel p, N = 64 x K = 32 channels, the FC
//       weights W[n, c*P2*P2 + p] (torch flattens [C, H, W]),
//       ((k/8)*8 + n/8)*64 + (n%8)*8 + k%8
//
// Warp roles (352 threads): warp 0 = producers (lane 0: cp.async.bulk of the
// conv1 pixel blocks, lane 1: the FC weight blocks; mbarrier complete_tx);
// warp 1 = TMEM allocator + conv2 MMA issuer and warp 10 = FC MMA issuer (each
// warp runs its loop, an elected lane issues its tcgen05.mma/commit); warps
// 2..9 = two epilogue groups (alternate output rows; tcgen05.ld of their TMEM
// lane quadrant, one env per thread).
//
// Traversal: output columns in chunks of CW = 7 (9 conv1 columns), output rows
// top to bottom, conv1 rows streaming through a 4-row ring in shared memory.
// tcgen05.mma costs >= 46 cycles per instruction for N <= 64 (tools/mma_rate.cu),
// so conv2 is issued with N = 96: conv1 block (row y+dy, column c) times the
// weights of the three taps (dy, 2), (dy, 1), (dy, 0) side by side lands on
// output pixels c-2, c-1, c of row y in one MMA (narrower at the chunk edges).
// One output row's 7 pixels are one accumulator row in TMEM (224 columns, two
// rows double-buffered); every MMA accumulates into accumulators the epilogue
// zeroes after reading them. 27 conv2 MMAs per 7 output pixels instead of 63.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "env_kernels.cuh"  // splitmix64

namespace lg {
namespace tc {

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// A pipeline bug must not hang the GPU: after ~2^31 cycles (> 1 s) of waiting
// on one phase the kernel traps (the launch fails with an error instead).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try(bar, parity)) {
        if (clock64() - t0 > (1ll << 31)) __trap();
    }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .b32 r;\n.reg .pred p;\nelect.sync r|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory matrix descriptor, K-major, no swizzle: start address,
// leading (K-direction core-matrix) and stride (M/N-direction) byte offsets,
// descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// A operand from TMEM (a_tmem: 128 lanes x 8 columns per K = 16 step), B from shared memory
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// shared memory (UMMA descriptor) -> TMEM, 128 rows x 256 bits: one 128 x 16 bf16 block
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// 32 lanes x 32 consecutive columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// zero 32 consecutive columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_zero32(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 16 registers -> 16 consecutive columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// a float in the shared memory of CTA `rank` of the cluster (same offset as `local`)
__device__ __forceinline__ float ld_peer_f32(const void *local, uint32_t rank) {
    uint32_t ra;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(local)), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}

}  // namespace tc

struct TrunkParams {
    const __nv_bfloat16 *c1;  // conv1 tiles (layout above)
    const __nv_bfloat16 *w2;  // [9][512]
    const float *b2;          // [32]
    const __nv_bfloat16 *w3;  // [P2*P2][2048]
    const float *b3;          // [64]
    const float *wh;          // [NA + 1][64]: policy head rows, then the value head
    const float *bh;          // [NA + 1]
    float *logits;            // [B][NA]
    float *value;             // [B]
    long long B;
    long long tile0;          // first 128-env tile of this launch
    int P1, NA;
    // fused sampling (lg_policy_trunk_sample): a ~ Categorical(logits) per env
    long long *actions;       // [B] or null
    float *logp;              // [B]: log pi(a) (ppo.py:128-130)
    unsigned long long seed;  // counter-based draw per (seed, env)
};

#ifdef TK_PROF  // cycle accounting of the MMA issuer and one epilogue thread (tools/trunk_prof.py)
__device__ long long g_tk_prof[1024][16];
#define TKP(k, v) (prof[k] += (v))
#else
#define TKP(k, v)
#endif
#ifndef TK_CHUNK
#define TK_CHUNK 7
#endif
constexpr int TK_CW = TK_CHUNK;               // output columns per chunk
constexpr int TK_RC = TK_CW + 2;              // conv1 columns per ring row
constexpr int TK_RING = 4;                    // conv1 rows in shared memory
#ifndef TK_W3_SLOTS
#define TK_W3_SLOTS 8
#endif
#ifndef TK_A3_SLOTS
#define TK_A3_SLOTS 2
#endif
constexpr int TK_W3 = TK_W3_SLOTS;            // FC weight blocks in flight (released in pairs)
constexpr int TK_EPI = 2;                     // epilogue warp groups (output row R -> group R % 2)
#ifndef TK_A3_TMEM
#define TK_A3_TMEM 0  // extra FC A-operand slots per group kept in TMEM (16 columns each, TS MMAs)
#endif
constexpr int TK_A3S = TK_A3_SLOTS;           // conv2 activation blocks in shared memory per group
constexpr int TK_A3G = TK_A3_SLOTS + TK_A3_TMEM;  // activation slots (FC A operand) per group
constexpr int TK_THREADS = 64 + 128 * TK_EPI + 32;  // + the FC issuer warp
constexpr int TK_MAXNA = 16;
constexpr uint32_t TK_BLK = 4096;             // one 128 x 16 bf16 block
// TMEM columns: one conv2 accumulator row (CW pixels x 32 channels) per epilogue group + FC accumulator
constexpr uint32_t TK_T_ACC = 0;
constexpr uint32_t TK_T_D3 = TK_T_ACC + TK_EPI * TK_CW * 32;  // 448
constexpr uint32_t TK_T_A3 = TK_T_D3 + 64;                      // TMEM activation slots
static_assert(TK_T_A3 + TK_EPI * TK_A3_TMEM * 16 <= 512, "TMEM budget");
static_assert(TK_CW <= 7, "conv2_row dispatch covers chunk widths 1..7");
constexpr uint32_t TK_OFF_RING = 0;
constexpr uint32_t TK_OFF_W2 = TK_OFF_RING + TK_RING * TK_RC * TK_BLK;  // 147456: 3 x [96 x 16] bf16
constexpr uint32_t TK_OFF_W3 = TK_OFF_W2 + 3 * 3072;
constexpr uint32_t TK_OFF_A3 = TK_OFF_W3 + TK_W3 * 4096;
constexpr uint32_t TK_OFF_HEAD = TK_OFF_A3 + TK_EPI * TK_A3S * 8192;
constexpr uint32_t TK_OFF_BIAS = TK_OFF_HEAD + (TK_MAXNA + 1) * 64 * 4;
constexpr uint32_t TK_OFF_BAR = (TK_OFF_BIAS + (32 + 64 + TK_MAXNA + 1) * 4 + 7) & ~7u;  // 8-byte aligned
constexpr int TK_NBAR = 2 * TK_RING + TK_W3 + TK_W3 / 2 + 2 * TK_EPI + 2 * TK_EPI * TK_A3G + 2;
constexpr uint32_t TK_SMEM = TK_OFF_BAR + TK_NBAR * 8 + 16;
static_assert(TK_SMEM <= 227 * 1024, "shared memory budget");

// One output row's conv2 (CW pixels): conv1 block (row y+dy, column c) x the
// three taps (dy, 2..0) -> pixels c-2..c, N = 96 (narrower at the edges).
// Fully unrolled so every offset and instruction descriptor is an immediate.
template <int CW>
__device__ __forceinline__ void conv2_row(uint32_t acc, const uint64_t (&dr)[3], uint64_t d_w2) {
#pragma unroll
    for (int dy = 0; dy < 3; dy++) {
#pragma unroll
        for (int c = 0; c < CW + 2; c++) {
            const int xlo = c - 2 > 0 ? c - 2 : 0, xhi = c < CW - 1 ? c : CW - 1;
            const int jb = xlo - c + 2, n = 32 * (xhi - xlo + 1);
            tc::mma_bf16(acc + 32u * xlo, dr[dy] + ((uint32_t)c * TK_BLK >> 4),
                         d_w2 + ((uint32_t)(dy * 3072 + jb * 512) >> 4), tc::idesc_bf16(128, n), 1u);
        }
    }
}

// bias + ReLU of the FC accumulator row, then the policy and value heads
// (fp32), and with p.actions the action draw of ppo.py:125-130
__device__ __forceinline__ void trunk_heads(const TrunkParams &p, const float *head, const float *bias3,
                                            const float *biash, float (&h)[64], long long env) {
#pragma unroll
    for (int j = 0; j < 64; j++) {
        const float v = h[j] + bias3[j];
        h[j] = v > 0.f ? v : 0.f;
    }
    if (env >= p.B) return;
    float lg[TK_MAXNA];
    float mx = -INFINITY;
    for (int o = 0; o <= p.NA; o++) {
        const float *wr = head + o * 64;
        float a = biash[o];
#pragma unroll
        for (int j = 0; j < 64; j++) a = fmaf(h[j], wr[j], a);
        if (o < p.NA) {
            p.logits[env * p.NA + o] = a;
            if (p.actions) {
#pragma unroll
                for (int q = 0; q < TK_MAXNA; q++)
                    if (q == o) lg[q] = a;  // register array: static indices only
                mx = fmaxf(mx, a);
            }
        } else {
            p.value[env] = a;
        }
    }
    if (p.actions) {  // Categorical(logits).sample() and its log-probability
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < TK_MAXNA; q++)
            if (q < p.NA) sum += __expf(lg[q] - mx);
        const uint64_t x = splitmix64(p.seed * 0xD1B54A32D192ED03ULL ^ splitmix64((uint64_t)env));
        const float u = (float)(x >> 40) * (1.0f / 16777216.0f) * sum;
        float c = 0.f, la = lg[0];
        int a = 0;
#pragma unroll
        for (int q = 0; q < TK_MAXNA; q++) {
            if (q < p.NA) {
                c += __expf(lg[q] - mx);
                if (c <= u && q + 1 < p.NA) {
                    a = q + 1;
                    la = lg[q + 1];
                }
            }
        }
        p.actions[env] = a;
        p.logp[env] = la - mx - __logf(sum);
    }
}

// SPLIT: launched in clusters of 2 for the tail of a launch (the tiles past
// its last whole wave): the two CTAs of a cluster take the two halves of one
// tile's column chunks, each accumulates its pixels' FC partial sums in its
// own TMEM, CTA 1 hands its partial to CTA 0 through distributed shared
// memory, and CTA 0 finishes the heads. 512 tiles (65,536 envs) on 148 SMs
// are 3 whole waves + 68 tiles: the 68 run as 136 half-tile CTAs in one
// wave of roughly half a tile's time instead of a fourth whole-tile wave.
template <bool SPLIT>
__global__ void __launch_bounds__(TK_THREADS, 1) trunk_kernel_t(const TrunkParams p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P1 = p.P1, P2 = P1 - 2, NP1 = P1 * P1;
    const int nch_all = (P2 + TK_CW - 1) / TK_CW;
    const int rank = SPLIT ? (int)tc::cluster_rank() : 0;
    const int cxa = SPLIT ? rank * ((nch_all + 1) / 2) : 0;  // this CTA's column chunks
    const int cxb = SPLIT && rank == 0 ? (nch_all + 1) / 2 : nch_all;
    const int nrows = (cxb - cxa) * P2;  // output rows over this CTA's chunks
    const long long tile = p.tile0 + (SPLIT ? blockIdx.x / 2 : blockIdx.x);
    const uint32_t s0 = tc::su32(sm);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + TK_OFF_BAR);
    const uint32_t b0 = tc::su32(bars);
    auto BAR = [&](int i) { return b0 + 8u * (uint32_t)i; };
    // barrier ids
    const int C1F = 0, C1E = C1F + TK_RING, W3F = C1E + TK_RING, W3E = W3F + TK_W3, ACF = W3E + TK_W3 / 2,
              ACE = ACF + TK_EPI, A3F = ACE + TK_EPI, A3E = A3F + TK_EPI * TK_A3G, D3F = A3E + TK_EPI * TK_A3G,
              W2F = D3F + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + TK_OFF_BAR + TK_NBAR * 8);
    float *head = reinterpret_cast<float *>(sm + TK_OFF_HEAD);
    float *bias2 = reinterpret_cast<float *>(sm + TK_OFF_BIAS), *bias3 = bias2 + 32, *biash = bias3 + 64;

    if (threadIdx.x == 0) {
        for (int i = 0; i < TK_RING; i++) tc::mbar_init(BAR(C1F + i), 1), tc::mbar_init(BAR(C1E + i), 1);
        for (int i = 0; i < TK_W3; i++) tc::mbar_init(BAR(W3F + i), 1);
        for (int i = 0; i < TK_W3 / 2; i++) tc::mbar_init(BAR(W3E + i), 1);
        for (int i = 0; i < TK_EPI; i++) tc::mbar_init(BAR(ACF + i), 1), tc::mbar_init(BAR(ACE + i), 128);
        for (int i = 0; i < TK_EPI * TK_A3G; i++) tc::mbar_init(BAR(A3F + i), 128), tc::mbar_init(BAR(A3E + i), 1);
        tc::mbar_init(BAR(D3F), 1);
        tc::mbar_init(BAR(W2F), 1);
        tc::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < (p.NA + 1) * 64; i += blockDim.x) head[i] = p.wh[i];
    for (int i = threadIdx.x; i < 32; i += blockDim.x) bias2[i] = p.b2[i];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) bias3[i] = p.b3[i];
    for (int i = threadIdx.x; i < p.NA + 1; i += blockDim.x) biash[i] = p.bh[i];
    if (warp == 1) {  // TMEM: two conv2 accumulator rows + the FC accumulator (512 columns)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::su32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc::tc_before();
    __syncthreads();
    tc::tc_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t T_D3 = tmem + TK_T_D3;

    if (warp == 0) {
        // ---------------- producers: lane 0 streams the conv1 rows, lane 1 the
        // FC weight blocks (independent threads, so neither stream can block
        // the other: a row's FCs are issued after the next row's conv2)
        if (lane == 0) {
            const uint8_t *c1 = reinterpret_cast<const uint8_t *>(p.c1) + (size_t)tile * NP1 * TK_BLK;
            tc::mbar_expect_tx(BAR(W2F), 3 * 3072);
            tc::bulk_g2s(s0 + TK_OFF_W2, p.w2, 3 * 3072, BAR(W2F));
            int L = 0;
            for (int cx = cxa; cx < cxb; cx++) {
                const int ncol = min(TK_RC, P1 - cx * TK_CW);
                for (int r = 0; r < P1; r++, L++) {
                    const int slot = L % TK_RING;
                    if (L >= TK_RING) tc::mbar_wait(BAR(C1E + slot), (uint32_t)((L / TK_RING - 1) & 1));
                    tc::mbar_expect_tx(BAR(C1F + slot), (uint32_t)ncol * TK_BLK);
                    for (int j = 0; j < ncol; j++)
                        tc::bulk_g2s(s0 + TK_OFF_RING + (uint32_t)(slot * TK_RC + j) * TK_BLK,
                                     c1 + (size_t)(r * P1 + cx * TK_CW + j) * TK_BLK, TK_BLK, BAR(C1F + slot));
                }
            }
        } else if (lane == 1) {
            const uint8_t *w3 = reinterpret_cast<const uint8_t *>(p.w3);
            int pix = 0;
            for (int cx = cxa; cx < cxb; cx++) {
                const int cw = min(TK_CW, P2 - cx * TK_CW);
                for (int y = 0; y < P2; y++)
                    for (int xl = 0; xl < cw; xl++, pix++) {
                        const int slot = pix % TK_W3;
                        if (pix >= TK_W3 && (slot & 1) == 0)  // slots are released in pairs
                            tc::mbar_wait(BAR(W3E + slot / 2), (uint32_t)((pix / TK_W3 - 1) & 1));
                        tc::mbar_expect_tx(BAR(W3F + slot), 4096);
                        tc::bulk_g2s(s0 + TK_OFF_W3 + slot * 4096u,
                                     w3 + (size_t)(y * P2 + cx * TK_CW + xl) * 4096, 4096, BAR(W3F + slot));
                    }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: the whole warp runs the loop (warp-uniform
        // values stay in uniform registers), one elected lane issues ----------------
#ifdef TK_PROF
        long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tq = clock64(), t0 = tq;
#define TKT(k)                          \
    do {                                \
        const long long _t = clock64(); \
        TKP(k, _t - tq);                \
        tq = _t;                        \
    } while (0)
#else
#define TKT(k)
#endif
        tc::mbar_wait(BAR(W2F), 0);
        // descriptor bases; a shared-memory offset is added as (bytes >> 4)
        const uint64_t d_ring = tc::sdesc(s0 + TK_OFF_RING, 2048, 128);
        const uint64_t d_w2 = tc::sdesc(s0 + TK_OFF_W2, 1536, 128);
        int Lw = 0;   // conv1 rows waited for
        int R = 0;
        for (int cx = cxa; cx < cxb; cx++) {
            const int cw = min(TK_CW, P2 - cx * TK_CW);
            const int L0 = (cx - cxa) * P1;  // ring rows this CTA streamed before chunk cx
            for (int y = 0; y < P2; y++, R++) {
                const int ab = R % TK_EPI;
                TKT(0);
                tc::mbar_wait(BAR(ACE + ab), (uint32_t)((R / TK_EPI) & 1));  // zeroed, drained
                TKT(3);
                for (; Lw <= L0 + y + 2; Lw++) tc::mbar_wait(BAR(C1F + Lw % TK_RING), (uint32_t)((Lw / TK_RING) & 1));
                TKT(4);
                tc::tc_after();
                const uint32_t acc = tmem + TK_T_ACC + (uint32_t)ab * (TK_CW * 32);
                const uint64_t dr[3] = {d_ring + ((uint32_t)(((L0 + y) % TK_RING) * TK_RC) * TK_BLK >> 4),
                                        d_ring + ((uint32_t)(((L0 + y + 1) % TK_RING) * TK_RC) * TK_BLK >> 4),
                                        d_ring + ((uint32_t)(((L0 + y + 2) % TK_RING) * TK_RC) * TK_BLK >> 4)};
                if (tc::elect_one()) {
                    switch (cw) {
                    case 7: conv2_row<7>(acc, dr, d_w2); break;
                    case 6: conv2_row<6>(acc, dr, d_w2); break;
                    case 5: conv2_row<5>(acc, dr, d_w2); break;
                    case 4: conv2_row<4>(acc, dr, d_w2); break;
                    case 3: conv2_row<3>(acc, dr, d_w2); break;
                    case 2: conv2_row<2>(acc, dr, d_w2); break;
                    default: conv2_row<1>(acc, dr, d_w2); break;
                    }
                    tc::mma_commit(BAR(ACF + ab));
                    tc::mma_commit(BAR(C1E + (L0 + y) % TK_RING));  // conv1 row y is no longer read
                    if (y == P2 - 1) {
                        tc::mma_commit(BAR(C1E + (L0 + P2) % TK_RING));
                        tc::mma_commit(BAR(C1E + (L0 + P2 + 1) % TK_RING));
                    }
                }
                __syncwarp();
                TKT(5);
            }
        }
#ifdef TK_PROF
        TKT(0);
        prof[7] = clock64() - t0;
        if (lane == 0)
            for (int k2 = 0; k2 < 8; k2++) g_tk_prof[blockIdx.x & 1023][k2] = prof[k2];
#endif
    } else if (warp == 2 + 4 * TK_EPI) {
        // ---------------- FC issuer: a second MMA-issuing warp, so the FC's
        // waits (epilogue activations, weight blocks) and commits never stall the
        // conv2 issue (tcgen05.commit tracks the issuing thread's own MMAs) ----------------
        constexpr uint32_t ID3 = tc::idesc_bf16(128, 64);
        const uint64_t d_a3 = tc::sdesc(s0 + TK_OFF_A3, 2048, 128);
        const uint64_t d_w3 = tc::sdesc(s0 + TK_OFF_W3, 1024, 128);
        int pix = 0, kg0 = 0, kg1 = 0, R = 0;  // FC pixels issued; A3 blocks consumed per epilogue group
        for (int cx = cxa; cx < cxb; cx++) {
            const int cw = min(TK_CW, P2 - cx * TK_CW);
            for (int y = 0; y < P2; y++, R++) {
                const int g = R % TK_EPI;
                int &kg = g ? kg1 : kg0;
                for (int j = 0; j < cw; j++, pix++, kg++) {  // D3 += relu(conv2)(pixel) x W3(pixel)
                    const int sl = kg % TK_A3G, a = g * TK_A3G + sl, w = pix % TK_W3;
                    tc::mbar_wait(BAR(A3F + a), (uint32_t)((kg / TK_A3G) & 1));
                    tc::mbar_wait(BAR(W3F + w), (uint32_t)((pix / TK_W3) & 1));
                    tc::tc_after();
                    if (tc::elect_one()) {
                        if (TK_A3_TMEM == 0 || sl < TK_A3S) {  // A from shared memory
                            const uint32_t as = (uint32_t)(g * TK_A3S + sl) * 8192u;
                            tc::mma_bf16(T_D3, d_a3 + (as >> 4), d_w3 + ((uint32_t)w * 4096u >> 4), ID3,
                                         pix > 0 ? 1u : 0u);
                            tc::mma_bf16(T_D3, d_a3 + ((as + 4096u) >> 4), d_w3 + (((uint32_t)w * 4096u + 2048u) >> 4),
                                         ID3, 1u);
                        } else {  // A from TMEM: 16 columns, channels (2c, 2c + 1) in column c
                            const uint32_t at = tmem + TK_T_A3 + 16u * (uint32_t)(g * TK_A3_TMEM + sl - TK_A3S);
                            tc::mma_bf16_ts(T_D3, at, d_w3 + ((uint32_t)w * 4096u >> 4), ID3, pix > 0 ? 1u : 0u);
                            tc::mma_bf16_ts(T_D3, at + 8u, d_w3 + (((uint32_t)w * 4096u + 2048u) >> 4), ID3, 1u);
                        }
                        tc::mma_commit(BAR(A3E + a));
                        if (w & 1) tc::mma_commit(BAR(W3E + w / 2));
                    }
                    __syncwarp();
                }
            }
        }
        if (tc::elect_one()) tc::mma_commit(BAR(D3F));
        __syncwarp();
    } else {  // ---------------- epilogue: TK_EPI groups of 4 warps, one env (TMEM lane) per thread ----------------
        const int grp = (warp - 2) >> 2;  // output row R is handled by group R % TK_EPI
        const int q = warp & 3;           // TMEM lane quadrant this warp may access
        const int m = q * 32 + lane;      // env row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const uint32_t acc = tmem + TK_T_ACC + lane_off + (uint32_t)grp * (TK_CW * 32);
        float b2r[32];
#pragma unroll
        for (int c = 0; c < 32; c++) b2r[c] = bias2[c];
        // the accumulators start at zero (every conv2 MMA accumulates)
        for (int j = 0; j < TK_CW; j++) tc::tmem_zero32(acc + 32u * j);
        tc::tmem_wait_st();
        tc::tc_before();
        tc::mbar_arrive(BAR(ACE + grp));
        int k = 0;  // A3 blocks produced by this group
#ifdef TK_PROF
        long long eprof[4] = {0, 0, 0, 0}, e0 = clock64();
#endif
        for (int R = grp; R < nrows; R += TK_EPI) {
            const int cw = min(TK_CW, P2 - (cxa + R / P2) * TK_CW);
#ifdef TK_PROF
            long long ew = clock64();
#endif
            tc::mbar_wait(BAR(ACF + grp), (uint32_t)((R / TK_EPI) & 1));
#ifdef TK_PROF
            eprof[0] += clock64() - ew;
#endif
            tc::tc_after();
            __syncwarp();
            for (int j = 0; j < cw; j++, k++) {
                uint32_t r[32];
                tc::tmem_ld32(acc + 32u * j, r);
                tc::tmem_wait_ld();
                tc::tmem_zero32(acc + 32u * j);
                const int sl = k % TK_A3G, a = grp * TK_A3G + sl;
#ifdef TK_PROF
                long long ea = clock64();
#endif
                if (k >= TK_A3G) tc::mbar_wait(BAR(A3E + a), (uint32_t)((k / TK_A3G - 1) & 1));
#ifdef TK_PROF
                eprof[1] += clock64() - ea;
#endif
                if (TK_A3_TMEM > 0 && sl >= TK_A3S) {  // TMEM slot: bf16 pairs, one column per two channels
                    uint32_t wd[16];
#pragma unroll
                    for (int c2 = 0; c2 < 16; c2++) {
                        float x0 = __uint_as_float(r[2 * c2]) + b2r[2 * c2];
                        float x1 = __uint_as_float(r[2 * c2 + 1]) + b2r[2 * c2 + 1];
                        x0 = x0 > 0.f ? x0 : 0.f;
                        x1 = x1 > 0.f ? x1 : 0.f;
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
                        wd[c2] = *reinterpret_cast<uint32_t *>(&h2);
                    }
                    tc::tmem_st16(tmem + lane_off + TK_T_A3 + 16u * (uint32_t)(grp * TK_A3_TMEM + sl - TK_A3S), wd);
                    tc::tmem_wait_st();
                    tc::tc_before();
                    tc::mbar_arrive(BAR(A3F + a));
                    __syncwarp();
                    continue;
                }
                uint8_t *a3 = sm + TK_OFF_A3 + (uint32_t)(grp * TK_A3S + sl) * 8192u;
#pragma unroll
                for (int kc = 0; kc < 4; kc++) {  // 8 channels -> one 16-byte core-matrix row
                    uint32_t wd[4];
#pragma unroll
                    for (int jj = 0; jj < 4; jj++) {
                        const int c = kc * 8 + 2 * jj;
                        float x0 = __uint_as_float(r[c]) + b2r[c], x1 = __uint_as_float(r[c + 1]) + b2r[c + 1];
                        x0 = x0 > 0.f ? x0 : 0.f;
                        x1 = x1 > 0.f ? x1 : 0.f;
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
                        wd[jj] = *reinterpret_cast<uint32_t *>(&h2);
                    }
                    *reinterpret_cast<uint4 *>(a3 + ((kc * 16 + (m >> 3)) * 128 + (m & 7) * 16)) =
                        make_uint4(wd[0], wd[1], wd[2], wd[3]);
                }
                tc::fence_proxy_async();
                tc::mbar_arrive(BAR(A3F + a));
                __syncwarp();
            }
            tc::tmem_wait_st();
            tc::tc_before();
            tc::mbar_arrive(BAR(ACE + grp));
        }
#ifdef TK_PROF
        if (threadIdx.x == 64 || threadIdx.x == 64 + 128) {
            eprof[2] = clock64() - e0;
            for (int k2 = 0; k2 < 3; k2++) g_tk_prof[blockIdx.x & 1023][8 + 4 * grp + k2] = eprof[k2];
        }
#endif
        if (grp == 0) {
            tc::mbar_wait(BAR(D3F), 0);
            tc::tc_after();
            __syncwarp();
            float h[64];
#pragma unroll
            for (int half = 0; half < 2; half++) {
                uint32_t r[32];
                tc::tmem_ld32(T_D3 + lane_off + half * 32, r);
                tc::tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j++) h[half * 32 + j] = __uint_as_float(r[j]);
            }
            if constexpr (!SPLIT) {
                trunk_heads(p, head, bias3, biash, h, tile * 128 + m);
            } else {  // the partial sums go to shared memory: [64][128] floats in the (idle) ring
                float *xb = reinterpret_cast<float *>(sm + TK_OFF_RING);
#pragma unroll
                for (int j = 0; j < 64; j++) xb[j * 128 + m] = h[j];
            }
        }
    }
    if constexpr (SPLIT) {
        tc::cluster_sync();  // both partials are in shared memory
        if (rank == 0 && warp >= 2 && warp < 6) {  // epilogue group 0 of CTA 0: sum, bias, ReLU, heads
            const int m = (warp & 3) * 32 + lane;
            const float *xb = reinterpret_cast<const float *>(sm + TK_OFF_RING);
            float h[64];
#pragma unroll
            for (int j = 0; j < 64; j++) h[j] = xb[j * 128 + m] + tc::ld_peer_f32(xb + j * 128 + m, 1);
            trunk_heads(p, head, bias3, biash, h, tile * 128 + m);
        }
        tc::cluster_sync();  // CTA 0 has read CTA 1's shared memory
    }
    tc::tc_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace lg
