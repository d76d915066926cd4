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
//   w2  [9 taps][512]: N = 32 out x K = 16 in, ((k/8)*4 + n/8)*64 + (n%8)*8 + k%8
//   w3  [P2*P2][2048]: per conv2 pixel p, N = 64 x K = 32 channels, the FC
//       weights W[n, c*P2*P2 + p] (torch flattens [C, H, W]),
//       ((k/8)*8 + n/8)*64 + (n%8)*8 + k%8
//
// Warp roles (320 threads): warp 0 = producers (lane 0: cp.async.bulk of the
// conv1 pixel blocks, lane 1: the FC weight blocks; mbarrier complete_tx);
// warp 1 = TMEM allocator + lane 0 issues every tcgen05.cp/mma/commit;
// warps 2..9 = two epilogue groups (alternate conv2 pixels; tcgen05.ld of
// their TMEM lane quadrant, one env per thread).
//
// Traversal: output columns in chunks of CW = 7 (9 conv1 columns), output
// rows top to bottom. conv1 rows land in shared memory (2-row staging ring)
// and are copied into a 4-row ring in TMEM (tcgen05.cp 128x256b per block):
// conv2's A operands are read from TMEM (the "TS" MMA form), so the tensor
// core's shared-memory reads per conv2 tap are the 1 KB weight block only,
// not the 4 KB activation block. Each conv1 block is loaded ~9/7 times and
// every tap's A operand is a TMEM address into the ring (no im2col copy).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

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
    int P1, NA;
};

constexpr int TK_CW = 7;                      // output columns per chunk
constexpr int TK_RC = TK_CW + 2;              // conv1 columns per ring row
constexpr int TK_SRING = 2;                   // conv1 rows staged in shared memory (bulk-copy landing)
constexpr int TK_TRING = 4;                   // conv1 rows resident in TMEM (conv2 A operands)
constexpr int TK_W3 = 8;                      // FC weight blocks in flight
constexpr int TK_A3 = 4;                      // conv2 activation blocks (FC A operand)
constexpr int TK_D2 = 4;                      // conv2 accumulator slots in TMEM (32 columns each)
constexpr int TK_LAG = 2;                     // FC of pixel i is issued after conv2 of pixel i + LAG
constexpr int TK_EPI = 2;                     // epilogue warp groups (pixel i -> group i % 2)
constexpr int TK_THREADS = 64 + 128 * TK_EPI;
constexpr int TK_MAXNA = 16;
constexpr uint32_t TK_BLK = 4096;             // one 128 x 16 bf16 block
// TMEM columns: conv1 ring (8 per block), conv2 accumulators, FC accumulator
constexpr uint32_t TK_T_A = 0;
constexpr uint32_t TK_T_D2 = TK_T_A + TK_TRING * TK_RC * 8;  // 288
constexpr uint32_t TK_T_D3 = TK_T_D2 + TK_D2 * 32;           // 416
static_assert(TK_T_D3 + 64 <= 512, "TMEM budget");
static_assert(TK_D2 % TK_EPI == 0 && TK_A3 % TK_EPI == 0, "ring slots must map to one epilogue group");
constexpr uint32_t TK_OFF_RING = 0;
constexpr uint32_t TK_OFF_W2 = TK_OFF_RING + TK_SRING * TK_RC * TK_BLK;  // 73728
constexpr uint32_t TK_OFF_W3 = TK_OFF_W2 + 9 * 1024;
constexpr uint32_t TK_OFF_A3 = TK_OFF_W3 + TK_W3 * 4096;
constexpr uint32_t TK_OFF_HEAD = TK_OFF_A3 + TK_A3 * 8192;
constexpr uint32_t TK_OFF_BIAS = TK_OFF_HEAD + (TK_MAXNA + 1) * 64 * 4;
constexpr uint32_t TK_OFF_BAR = (TK_OFF_BIAS + (32 + 64 + TK_MAXNA + 1) * 4 + 7) & ~7u;  // 8-byte aligned
constexpr int TK_NBAR = 2 * TK_SRING + 2 * TK_W3 + 2 * TK_D2 + 2 * TK_A3 + 2;
constexpr uint32_t TK_SMEM = TK_OFF_BAR + TK_NBAR * 8 + 16;

__global__ void __launch_bounds__(TK_THREADS, 1) trunk_kernel(const TrunkParams p) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P1 = p.P1, P2 = P1 - 2, NP1 = P1 * P1, NP2 = P2 * P2;
    const int nch = (P2 + TK_CW - 1) / TK_CW;
    const long long tile = blockIdx.x;
    const uint32_t s0 = tc::su32(sm);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + TK_OFF_BAR);
    const uint32_t b0 = tc::su32(bars);
    auto BAR = [&](int i) { return b0 + 8u * (uint32_t)i; };
    // barrier ids
    const int C1F = 0, C1E = C1F + TK_SRING, W3F = C1E + TK_SRING, W3E = W3F + TK_W3, D2F = W3E + TK_W3,
              D2E = D2F + TK_D2, A3F = D2E + TK_D2, A3E = A3F + TK_A3, D3F = A3E + TK_A3, W2F = D3F + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + TK_OFF_BAR + TK_NBAR * 8);
    float *head = reinterpret_cast<float *>(sm + TK_OFF_HEAD);
    float *bias2 = reinterpret_cast<float *>(sm + TK_OFF_BIAS), *bias3 = bias2 + 32, *biash = bias3 + 64;

    if (threadIdx.x == 0) {
        for (int i = 0; i < TK_SRING; i++) tc::mbar_init(BAR(C1F + i), 1), tc::mbar_init(BAR(C1E + i), 1);
        for (int i = 0; i < TK_W3; i++) tc::mbar_init(BAR(W3F + i), 1), tc::mbar_init(BAR(W3E + i), 1);
        for (int i = 0; i < TK_D2; i++) tc::mbar_init(BAR(D2F + i), 1), tc::mbar_init(BAR(D2E + i), 128);
        for (int i = 0; i < TK_A3; i++) tc::mbar_init(BAR(A3F + i), 128), tc::mbar_init(BAR(A3E + i), 1);
        tc::mbar_init(BAR(D3F), 1);
        tc::mbar_init(BAR(W2F), 1);
        tc::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < (p.NA + 1) * 64; i += blockDim.x) head[i] = p.wh[i];
    for (int i = threadIdx.x; i < 32; i += blockDim.x) bias2[i] = p.b2[i];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) bias3[i] = p.b3[i];
    for (int i = threadIdx.x; i < p.NA + 1; i += blockDim.x) biash[i] = p.bh[i];
    if (warp == 1) {  // TMEM: conv1 ring + conv2 accumulators + FC accumulator (480 of 512 columns)
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
        // the other: the FC of a pixel is issued LAG pixels after its conv2)
        if (lane == 0) {
            const uint8_t *c1 = reinterpret_cast<const uint8_t *>(p.c1) + (size_t)tile * NP1 * TK_BLK;
            tc::mbar_expect_tx(BAR(W2F), 9 * 1024);
            tc::bulk_g2s(s0 + TK_OFF_W2, p.w2, 9 * 1024, BAR(W2F));
            int L = 0;
            for (int cx = 0; cx < nch; cx++) {
                const int ncol = min(TK_RC, P1 - cx * TK_CW);
                for (int r = 0; r < P1; r++, L++) {
                    const int slot = L % TK_SRING;
                    if (L >= TK_SRING) tc::mbar_wait(BAR(C1E + slot), (uint32_t)((L / TK_SRING - 1) & 1));
                    tc::mbar_expect_tx(BAR(C1F + slot), (uint32_t)ncol * TK_BLK);
                    for (int j = 0; j < ncol; j++)
                        tc::bulk_g2s(s0 + TK_OFF_RING + (uint32_t)(slot * TK_RC + j) * TK_BLK,
                                     c1 + (size_t)(r * P1 + cx * TK_CW + j) * TK_BLK, TK_BLK, BAR(C1F + slot));
                }
            }
        } else if (lane == 1) {
            const uint8_t *w3 = reinterpret_cast<const uint8_t *>(p.w3);
            int pix = 0;
            for (int cx = 0; cx < nch; cx++) {
                const int cw = min(TK_CW, P2 - cx * TK_CW);
                for (int y = 0; y < P2; y++)
                    for (int xl = 0; xl < cw; xl++, pix++) {
                        const int slot = pix % TK_W3;
                        if (pix >= TK_W3) tc::mbar_wait(BAR(W3E + slot), (uint32_t)((pix / TK_W3 - 1) & 1));
                        tc::mbar_expect_tx(BAR(W3F + slot), 4096);
                        tc::bulk_g2s(s0 + TK_OFF_W3 + slot * 4096u,
                                     w3 + (size_t)(y * P2 + cx * TK_CW + xl) * 4096, 4096, BAR(W3F + slot));
                    }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            constexpr uint32_t ID2 = tc::idesc_bf16(128, 32), ID3 = tc::idesc_bf16(128, 64);
            tc::mbar_wait(BAR(W2F), 0);
            int Lc = 0;  // conv1 rows copied into TMEM
            int pix = 0;
            auto fc = [&](int i) {  // D3 += relu(conv2)(pixel i) x W3(pixel i)
                const int a = i % TK_A3, w = i % TK_W3;
                tc::mbar_wait(BAR(A3F + a), (uint32_t)((i / TK_A3) & 1));
                tc::mbar_wait(BAR(W3F + w), (uint32_t)((i / TK_W3) & 1));
                tc::tc_after();
                const uint32_t aa = s0 + TK_OFF_A3 + a * 8192u, ww = s0 + TK_OFF_W3 + w * 4096u;
#pragma unroll
                for (int k = 0; k < 2; k++)
                    tc::mma_bf16(T_D3, tc::sdesc(aa + k * 4096u, 2048, 128), tc::sdesc(ww + k * 2048u, 1024, 128), ID3,
                                 (i > 0 || k > 0) ? 1u : 0u);
                tc::mma_commit(BAR(A3E + a));
                tc::mma_commit(BAR(W3E + w));
            };
            for (int cx = 0; cx < nch; cx++) {
                const int cw = min(TK_CW, P2 - cx * TK_CW);
                const int ncol = min(TK_RC, P1 - cx * TK_CW);
                const int L0 = cx * P1;
                for (int y = 0; y < P2; y++) {
                    // conv1 rows up to y + 2 into the TMEM ring: shared -> TMEM copies run
                    // in issue order with the MMAs, so the slot of row L - TK_TRING (last
                    // read by output row y - 2's MMAs, issued before) is free
                    for (; Lc <= L0 + y + 2; Lc++) {
                        const int ss = Lc % TK_SRING;
                        tc::mbar_wait(BAR(C1F + ss), (uint32_t)((Lc / TK_SRING) & 1));
                        tc::tc_after();
                        const uint32_t ta = tmem + TK_T_A + (uint32_t)((Lc % TK_TRING) * TK_RC) * 8u;
                        for (int j = 0; j < ncol; j++)
                            tc::tmem_cp_128x256b(ta + j * 8u,
                                                 tc::sdesc(s0 + TK_OFF_RING + (uint32_t)(ss * TK_RC + j) * TK_BLK,
                                                           2048, 128));
                        tc::mma_commit(BAR(C1E + ss));  // the shared slot is free once the copies land
                    }
                    for (int xl = 0; xl < cw; xl++, pix++) {
                        const int s = pix % TK_D2;
                        if (pix >= TK_D2) {
                            tc::mbar_wait(BAR(D2E + s), (uint32_t)((pix / TK_D2 - 1) & 1));
                            tc::tc_after();
                        }
#pragma unroll
                        for (int t = 0; t < 9; t++) {
                            const int dy = t / 3, dx = t % 3;
                            const uint32_t a_t =
                                tmem + TK_T_A + (uint32_t)(((L0 + y + dy) % TK_TRING) * TK_RC + xl + dx) * 8u;
                            tc::mma_bf16_ts(tmem + TK_T_D2 + s * 32, a_t,
                                            tc::sdesc(s0 + TK_OFF_W2 + t * 1024u, 512, 128), ID2, t > 0 ? 1u : 0u);
                        }
                        tc::mma_commit(BAR(D2F + s));
                        if (pix >= TK_LAG) fc(pix - TK_LAG);
                    }
                }
            }
            for (int i = max(pix - TK_LAG, 0); i < pix; i++) fc(i);
            tc::mma_commit(BAR(D3F));
        }
    } else {  // ---------------- epilogue: TK_EPI groups of 4 warps, one env (TMEM lane) per thread ----------------
        const int grp = (warp - 2) >> 2;  // pixel i is handled by group i % TK_EPI
        const int q = warp & 3;           // TMEM lane quadrant this warp may access
        const int m = q * 32 + lane;      // env row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        float b2r[32];
#pragma unroll
        for (int c = 0; c < 32; c++) b2r[c] = bias2[c];
        for (int i = grp; i < NP2; i += TK_EPI) {
            const int s = i % TK_D2, a = i % TK_A3;
            tc::mbar_wait(BAR(D2F + s), (uint32_t)((i / TK_D2) & 1));
            tc::tc_after();
            uint32_t r[32];
            __syncwarp();
            tc::tmem_ld32(tmem + TK_T_D2 + lane_off + s * 32, r);
            tc::tmem_wait_ld();
            tc::tc_before();
            tc::mbar_arrive(BAR(D2E + s));
            if (i >= TK_A3) tc::mbar_wait(BAR(A3E + a), (uint32_t)((i / TK_A3 - 1) & 1));
            uint8_t *a3 = sm + TK_OFF_A3 + a * 8192u;
#pragma unroll
            for (int kc = 0; kc < 4; kc++) {  // 8 channels -> one 16-byte core-matrix row
                uint32_t wd[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int c = kc * 8 + 2 * j;
                    float x0 = __uint_as_float(r[c]) + b2r[c], x1 = __uint_as_float(r[c + 1]) + b2r[c + 1];
                    x0 = x0 > 0.f ? x0 : 0.f;
                    x1 = x1 > 0.f ? x1 : 0.f;
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
                    wd[j] = *reinterpret_cast<uint32_t *>(&h2);
                }
                *reinterpret_cast<uint4 *>(a3 + ((kc * 16 + (m >> 3)) * 128 + (m & 7) * 16)) =
                    make_uint4(wd[0], wd[1], wd[2], wd[3]);
            }
            tc::fence_proxy_async();
            tc::mbar_arrive(BAR(A3F + a));
        }
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
                for (int j = 0; j < 32; j++) {
                    const float v = __uint_as_float(r[j]) + bias3[half * 32 + j];
                    h[half * 32 + j] = v > 0.f ? v : 0.f;
                }
            }
            const long long env = tile * 128 + m;
            if (env < p.B) {
                for (int o = 0; o <= p.NA; o++) {
                    const float *wr = head + o * 64;
                    float acc = biash[o];
#pragma unroll
                    for (int j = 0; j < 64; j++) acc = fmaf(h[j], wr[j], acc);
                    if (o < p.NA) p.logits[env * p.NA + o] = acc;
                    else p.value[env] = acc;
                }
            }
        }
    }
    tc::tc_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace lg
