// solo.cuh -- one environment per THREAD for maps up to 16 x 16.
//
// A 16x16 bit-plane is eight 32-bit registers: word k holds row 2k in bits
// 0..15 and row 2k+1 in bits 16..31, so the bit index word*32+bit equals the
// row-major cell index r*16+c (np.argmax / flatnonzero order). A BFS layer is
// ~9 integer ops per word with no shuffles or votes: horizontal neighbours are
// in-word shifts (masked at the 16-bit row seam), vertical neighbours are one
// funnel shift with the adjacent word. 32 environments advance per warp with
// fully coalesced state loads; divergence (only ~1/3 of env-steps recompute
// metrics) costs far less than the collective traffic of a lane team.
#pragma once
#include <stdint.h>

#include "team.cuh"

namespace lg {

struct SB {
    uint32_t w[8];
    __device__ __forceinline__ static SB zero() {
        SB b;
#pragma unroll
        for (int k = 0; k < 8; k++) b.w[k] = 0;
        return b;
    }
    __device__ __forceinline__ bool nz() const {
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) x |= w[k];
        return x != 0;
    }
    __device__ __forceinline__ int count() const {
        int c = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) c += __popc(w[k]);
        return c;
    }
    // 16-bit row r (r static after unrolling, or dynamic). The word is picked
    // with AND/OR masks: a select chain is pattern-matched into a dynamically
    // indexed array, which demotes the plane to local memory.
    __device__ __forceinline__ uint32_t row(int r) const {
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) x |= w[k] & (0u - (uint32_t)(k == (r >> 1)));
        return (r & 1) ? (x >> 16) : (x & 0xFFFFu);
    }
};

__device__ __forceinline__ SB operator&(const SB &a, const SB &b) {
    SB o;
#pragma unroll
    for (int k = 0; k < 8; k++) o.w[k] = a.w[k] & b.w[k];
    return o;
}
__device__ __forceinline__ SB operator|(const SB &a, const SB &b) {
    SB o;
#pragma unroll
    for (int k = 0; k < 8; k++) o.w[k] = a.w[k] | b.w[k];
    return o;
}
__device__ __forceinline__ SB andnot(const SB &a, const SB &b) {
    SB o;
#pragma unroll
    for (int k = 0; k < 8; k++) o.w[k] = a.w[k] & ~b.w[k];
    return o;
}

__device__ __forceinline__ uint32_t mask16(int n) { return n >= 16 ? 0xFFFFu : ((1u << n) - 1u); }

// active rectangle h x w anchored top-left (apply_shape, grid.py:129-142)
__device__ __forceinline__ SB rect_sb(int h, int w) {
    SB b;
    uint32_t m = mask16(w);
#pragma unroll
    for (int k = 0; k < 8; k++) b.w[k] = ((2 * k < h) ? m : 0u) | ((2 * k + 1 < h) ? (m << 16) : 0u);
    return b;
}

__device__ __forceinline__ SB dilate_sb(const SB &f) {
    SB o;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint32_t x = f.w[k];
        uint32_t up = __funnelshift_l(k > 0 ? f.w[k - 1] : 0u, x, 16);  // row above
        uint32_t dn = __funnelshift_r(x, k < 7 ? f.w[k + 1] : 0u, 16);  // row below
        o.w[k] = x | ((x << 1) & 0xFFFEFFFEu) | ((x >> 1) & 0x7FFF7FFFu) | up | dn;
    }
    return o;
}

// Backend of the generic metric code (env_kernels.cuh) for one env per thread.
struct SoloK {
    using B = SB;
    static constexpr bool kIncRegions = false;  // register region count: cheap already
    __device__ __forceinline__ int regions_delta(const SB &, int, int, bool) const { return 0; }
    __device__ __forceinline__ int count(const SB &b) const { return b.count(); }
    __device__ __forceinline__ SB cell(int flat) const {
        SB b;
#pragma unroll
        for (int k = 0; k < 8; k++) b.w[k] = (k == (flat >> 5)) ? (1u << (flat & 31)) : 0u;
        return b;
    }
    __device__ __forceinline__ int kth(const SB &m, int kk) const {
        int res = 0;
        bool found = false;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            int c = __popc(m.w[k]);
            if (!found && kk < c) {
                uint32_t x = m.w[k];
                for (int i = 0; i < kk; i++) x &= x - 1;
                res = k * 32 + __ffs((int)x) - 1;
                found = true;
            }
            kk -= c;
        }
        return res;
    }
    __device__ __forceinline__ int lowest(const SB &m) const {
        int res = 0;
        bool found = false;
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (!found && m.w[k]) {
                res = k * 32 + __ffs((int)m.w[k]) - 1;
                found = true;
            }
        return res;
    }
    __device__ __forceinline__ int bfs_last(SB &f, const SB &pass) const {
        SB vis = f;
        int depth = 0;
        while (true) {
            SB nx = andnot(dilate_sb(f) & pass, vis);
            if (!nx.nz()) return depth;
            vis = vis | nx;
            f = nx;
            depth++;
        }
    }
    template <bool ENDPOINT>
    __device__ __forceinline__ void touch(SB f, const SB &pass, const SB &ta, const SB &tb, bool want_b, int &da,
                          int &db) const {
        da = -1;
        db = -1;
        bool need_a = ta.nz();
        bool need_b = want_b && tb.nz();
        SB vis = f;
        int depth = 0;
        while (need_a || need_b) {
            SB d = dilate_sb(f);
            if (ENDPOINT) {
                if (need_a && (d & ta).nz()) {
                    da = depth + 1;
                    need_a = false;
                }
                if (need_b && (d & tb).nz()) {
                    db = depth + 1;
                    need_b = false;
                }
            } else {
                if (need_a && (f & ta).nz()) {
                    da = depth;
                    need_a = false;
                }
                if (need_b && (f & tb).nz()) {
                    db = depth;
                    need_b = false;
                }
            }
            if (!need_a && !need_b) break;
            SB nx = andnot(d & pass, vis);
            if (!nx.nz()) break;
            vis = vis | nx;
            f = nx;
            depth++;
        }
    }
    // count_regions (pathfind.py:116-130) as a one-pass run labelling held in
    // registers: runs of set bits are nodes; only the runs of the previous row
    // (the frontier) can still merge, so each keeps a component label (byte k
    // of P0/P1 = label of run k) and a merge relabels the frontier with four
    // byte-wise compare-selects. regions = runs - merges of distinct labels,
    // the same count a union-find gives, without shared memory.
    __device__ __forceinline__ static uint32_t lab(uint32_t L0, uint32_t L1, int k) {
        return __byte_perm(L0, L1, (uint32_t)k) & 0xFFu;  // byte k of L1:L0
    }
    __device__ __forceinline__ static uint32_t relabel(uint32_t w, uint32_t from4, uint32_t to4) {
        const uint32_t m = __vcmpeq4(w, from4);
        return (w & ~m) | (to4 & m);
    }
    __device__ __forceinline__ int regions(const SB &pass, void *) const {
        int runs = 0, merges = 0;
        uint32_t prevR = 0, prevS = 0, P0 = 0, P1 = 0;
        // rolled row loop (instruction-cache footprint); the plane is shifted
        // down one row per iteration so the current row is always word 0's low half
        SB q = pass;
#pragma unroll 1
        for (int r = 0; r < 16; r++) {
            uint32_t R = q.w[0] & 0xFFFFu;
#pragma unroll
            for (int k = 0; k < 7; k++) q.w[k] = __funnelshift_r(q.w[k], q.w[k + 1], 16);
            q.w[7] >>= 16;
            uint32_t S = R & ~(R << 1);
            runs += __popc(S);
            // fresh label r*8 + k for run k of this row (<= 127, one byte)
            uint32_t C0 = (uint32_t)(r * 8) * 0x01010101u + 0x03020100u;
            uint32_t C1 = C0 + 0x04040404u;
            uint32_t C = R & prevR;
            uint32_t CS = C & ~(C << 1);  // one bit per (new run, old run) contact
            while (CS) {
                int c = __ffs((int)CS) - 1;
                CS &= CS - 1;
                uint32_t upto = (2u << c) - 1u;
                int ir = __popc(S & upto) - 1, ia = __popc(prevS & upto) - 1;
                uint32_t lc = lab(C0, C1, ir), la = lab(P0, P1, ia);
                if (lc == la) continue;
                merges++;
                if (lc >= (uint32_t)(r * 8)) {
                    // first contact of run ir: its fresh label occurs nowhere
                    // else, so only byte ir changes (to the old run's label)
                    const uint32_t j = (uint32_t)ir & 3u, sel = 0x3210u + ((4u - j) << (4u * j));
                    if (ir < 4) C0 = __byte_perm(C0, la, sel);
                    else C1 = __byte_perm(C1, la, sel);
                } else {  // two frontier components meet: relabel the larger id
                    const uint32_t hi4 = max(lc, la) * 0x01010101u, lo4 = min(lc, la) * 0x01010101u;
                    C0 = relabel(C0, hi4, lo4);
                    C1 = relabel(C1, hi4, lo4);
                    P0 = relabel(P0, hi4, lo4);
                    P1 = relabel(P1, hi4, lo4);
                }
            }
            P0 = C0;
            P1 = C1;
            prevR = R;
            prevS = S;
        }
        return runs - merges;
    }
};

}  // namespace lg
