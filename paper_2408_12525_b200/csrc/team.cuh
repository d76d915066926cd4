// team.cuh -- one environment per lane team: bit-packed rows + warp collectives.
//
// A "team" of TEAM lanes (16 or 32, a warp or half a warp) owns one
// environment. Lane l holds rows [l*RPL, l*RPL+RPL) of every bit-plane of the
// max grid as machine words (bit c = column c). All grid algorithms are then
// word-parallel per row and shuffle/vote-parallel across rows:
//   * BFS layer  = row dilation (shift by one bit, shuffle one lane up/down)
//                  masked by the passable plane (replaces the reference's
//                  max-filter fixpoint, pathfind.py:143-175);
//   * any/sum    = __any_sync / __reduce_add_sync over the team mask;
//   * regions    = run-based union-find in shared memory (count_regions,
//                  pathfind.py:116-130, same count).
#pragma once
#include <stdint.h>

// Debug builds (-DLG_CHECKS, tools/sanitize_cases.py): shared-memory index
// bounds are checked on device and a violation traps the launch. compute-
// sanitizer is closed on this GPU pool, so this is the out-of-bounds check.
#ifdef LG_CHECKS
#define LG_DCHECK(cond)         \
    do {                        \
        if (!(cond)) __trap();  \
    } while (0)
#else
#define LG_DCHECK(cond) \
    do {                \
    } while (0)
#endif

namespace lg {

template <int TEAM_, int RPL_, typename Row_, int MINB_ = 1>
struct Geo {
    static constexpr int MINB = MINB_;  // __launch_bounds__ min blocks (64-thread blocks) per SM
    static constexpr int TEAM = TEAM_;
    static constexpr int RPL = RPL_;
    static constexpr int ROWS = TEAM_ * RPL_;
    static constexpr int BITS = (int)sizeof(Row_) * 8;
    static constexpr int RUNS = BITS / 2;  // max runs of set bits in one row
    using Row = Row_;
};
using G16 = Geo<16, 1, uint32_t>;  // H <= 16, W <= 32
using G32 = Geo<32, 1, uint32_t>;  // H <= 32, W <= 32
// 64x64 maps are latency-bound (BFS shuffles, union-find): occupancy pays
// more than the spills of a 64-register budget (measured on c4, 32-thread
// blocks: 80 regs 84M, 64 regs 92M, 48 regs 91M env-steps/s).
#ifndef LG_G64_MINB
#define LG_G64_MINB 16
#endif
using G64 = Geo<32, 2, uint64_t, LG_G64_MINB>;  // H <= 64, W <= 64

__device__ __forceinline__ int ctz(uint32_t x) { return __ffs((int)x) - 1; }
__device__ __forceinline__ int ctz(uint64_t x) { return __ffsll((long long)x) - 1; }
__device__ __forceinline__ int msb(uint32_t x) { return 31 - __clz((int)x); }
__device__ __forceinline__ int msb(uint64_t x) { return 63 - __clzll((long long)x); }
__device__ __forceinline__ int popc(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc(uint64_t x) { return __popcll(x); }

template <typename Row>
__device__ __forceinline__ Row low_mask(int n) {
    constexpr int B = (int)sizeof(Row) * 8;
    return n >= B ? ~Row(0) : ((Row(1) << n) - Row(1));
}

template <class G>
struct Team {
    unsigned mask;  // lanes of this team within the warp
    int lane;       // 0..TEAM-1
    int base;       // first warp lane of the team
    __device__ __forceinline__ Team() {
        int l = threadIdx.x & 31;
        lane = l & (G::TEAM - 1);
        base = l - lane;
        mask = G::TEAM == 32 ? 0xffffffffu : (((1u << G::TEAM) - 1u) << base);
    }
    __device__ __forceinline__ int row(int k) const { return lane * G::RPL + k; }
    __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
    __device__ __forceinline__ unsigned ballot(bool p) const {
        return __ballot_sync(mask, p) >> base;
    }
    __device__ __forceinline__ int sum(int v) const {
        return (int)__reduce_add_sync(mask, (unsigned)v);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    template <typename T>
    __device__ __forceinline__ T from(T v, int src_lane) const {
        return __shfl_sync(mask, v, src_lane, G::TEAM);
    }
    // value held by lane-1 (0 for the first lane)
    template <typename T>
    __device__ __forceinline__ T up(T v) const {
        T r = __shfl_up_sync(mask, v, 1, G::TEAM);
        return lane == 0 ? T(0) : r;
    }
    // value held by lane+1 (0 for the last lane)
    template <typename T>
    __device__ __forceinline__ T down(T v) const {
        T r = __shfl_down_sync(mask, v, 1, G::TEAM);
        return lane == G::TEAM - 1 ? T(0) : r;
    }
    // inclusive prefix sum over lanes
    __device__ __forceinline__ int scan(int v) const {
#pragma unroll
        for (int o = 1; o < G::TEAM; o <<= 1) {
            int y = __shfl_up_sync(mask, v, o, G::TEAM);
            if (lane >= o) v += y;
        }
        return v;
    }
};

// The lane's slice of one bit-plane.
template <class G>
struct Bd {
    typename G::Row r[G::RPL];
    __device__ __forceinline__ static Bd zero() {
        Bd b;
#pragma unroll
        for (int k = 0; k < G::RPL; k++) b.r[k] = 0;
        return b;
    }
    __device__ __forceinline__ bool nz() const {
        typename G::Row x = 0;
#pragma unroll
        for (int k = 0; k < G::RPL; k++) x |= r[k];
        return x != 0;
    }
    __device__ __forceinline__ int count() const {
        int c = 0;
#pragma unroll
        for (int k = 0; k < G::RPL; k++) c += popc(r[k]);
        return c;
    }
};

#define LG_BD_OP(op)                                                              \
    template <class G>                                                            \
    __device__ __forceinline__ Bd<G> operator op(const Bd<G> &a, const Bd<G> &b) { \
        Bd<G> o;                                                                  \
        _Pragma("unroll") for (int k = 0; k < G::RPL; k++) o.r[k] = a.r[k] op b.r[k]; \
        return o;                                                                 \
    }
LG_BD_OP(&)
LG_BD_OP(|)
#undef LG_BD_OP

template <class G>
__device__ __forceinline__ Bd<G> andnot(const Bd<G> &a, const Bd<G> &b) {
    Bd<G> o;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) o.r[k] = a.r[k] & ~b.r[k];
    return o;
}

// Von Neumann dilation (cell plus its 4 neighbours), clipped to W columns.
template <class G>
__device__ __forceinline__ Bd<G> dilate(const Team<G> &t, const Bd<G> &f, typename G::Row wm) {
    Bd<G> o;
    if constexpr (G::RPL == 1) {
        auto a = t.up(f.r[0]);
        auto b = t.down(f.r[0]);
        o.r[0] = (f.r[0] | (f.r[0] << 1) | (f.r[0] >> 1) | a | b) & wm;
    } else {
        auto a = t.up(f.r[1]);    // row 2l-1
        auto b = t.down(f.r[0]);  // row 2l+2
        o.r[0] = (f.r[0] | (f.r[0] << 1) | (f.r[0] >> 1) | a | f.r[1]) & wm;
        o.r[1] = (f.r[1] | (f.r[1] << 1) | (f.r[1] >> 1) | f.r[0] | b) & wm;
    }
    return o;
}

// BFS from the cells of `f` through `pass`; on return `f` holds the last
// non-empty layer and the result is its depth (flood_distance layers).
// Two layers per team vote: layer 2 is non-empty only if layer 1 is, so one
// __any_sync decides both (half the votes and loop branches of a per-layer loop).
// (Four layers per vote measured slower on c4: 89 M -> 79 M env-steps/s, the
// extra live boards spill under the 64-register budget.)
template <class G>
__device__ __forceinline__ int bfs_last_layer(const Team<G> &t, Bd<G> &f, const Bd<G> &pass, typename G::Row wm) {
    Bd<G> vis = f;
    int depth = 0;
    while (true) {
        Bd<G> n1 = andnot(dilate(t, f, wm) & pass, vis);
        Bd<G> v1 = vis | n1;
        Bd<G> n2 = andnot(dilate(t, n1, wm) & pass, v1);
        if (!t.any(n2.nz())) {
            if (t.any(n1.nz())) {
                f = n1;
                depth++;
            }
            return depth;
        }
        vis = v1 | n2;
        f = n2;
        depth += 2;
    }
}

// First-touch distances of a BFS from `f` through `pass` to up to two target
// sets. ENDPOINT=false: first layer containing a target cell (raw distance,
// problems.py:190-191). ENDPOINT=true: targets are impassable endpoints read
// one step past their nearest reached neighbour (endpoint_field,
// pathfind.py:188-203), i.e. first layer whose dilation touches a target, +1.
// -1 = never touched.
// Two layers per round of votes: one ballot for "a target is touched in layer
// depth or depth+1" and one, independent of it (the two latencies overlap),
// for "layer depth+2 is non-empty"; an empty layer touches nothing and has
// only empty successors, so nothing is missed. The touched layer is resolved
// with extra votes once per target (c2 111 M -> 125 M env-steps/s vs one layer
// and two dependent votes per round).
template <class G, bool ENDPOINT>
__device__ __forceinline__ void bfs_touch(const Team<G> &t, Bd<G> f, const Bd<G> &pass, typename G::Row wm,
                          const Bd<G> &ta, const Bd<G> &tb, bool want_b, int &da, int &db) {
    da = -1;
    db = -1;
    bool need_a = t.any(ta.nz());
    bool need_b = want_b && t.any(tb.nz());
    Bd<G> vis = f;
    int depth = 0;
    constexpr int e = ENDPOINT ? 1 : 0;
    while (need_a || need_b) {
        Bd<G> d1 = dilate(t, f, wm);
        Bd<G> n1 = andnot(d1 & pass, vis);
        Bd<G> v1 = vis | n1;
        Bd<G> d2 = dilate(t, n1, wm);
        Bd<G> n2 = andnot(d2 & pass, v1);
        const Bd<G> &x0 = ENDPOINT ? d1 : f;   // touches layer `depth`
        const Bd<G> &x1 = ENDPOINT ? d2 : n1;  // touches layer `depth + 1`
        bool ha0 = need_a && (x0 & ta).nz(), ha1 = need_a && (x1 & ta).nz();
        bool hb0 = need_b && (x0 & tb).nz(), hb1 = need_b && (x1 & tb).nz();
        unsigned hit = t.ballot(ha0 | ha1 | hb0 | hb1);
        unsigned more = t.ballot(n2.nz());
        if (hit) {
            if (need_a && t.any(ha0 | ha1)) {
                da = depth + e + (t.any(ha0) ? 0 : 1);
                need_a = false;
            }
            if (need_b && t.any(hb0 | hb1)) {
                db = depth + e + (t.any(hb0) ? 0 : 1);
                need_b = false;
            }
        }
        if (!more) break;
        vis = v1 | n2;
        f = n2;
        depth += 2;
    }
}

// ---- run-based union-find region count -----------------------------------
// Nodes are runs of set bits, id = row * RUNS + run index (ids grow with the
// row, so links always point to smaller ids: ECL-CC style lock-free hooking).

__device__ __forceinline__ int uf_find(volatile uint16_t *par, int x) {
    int cur = par[x];
    if (cur != x) {
        int prev = x, next;
        while (cur > (next = par[cur])) {
            par[prev] = (uint16_t)next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

// returns 1 when two distinct trees were merged
__device__ __forceinline__ int uf_unite(volatile uint16_t *par, int a, int b) {
    int ra = uf_find(par, a), rb = uf_find(par, b);
    while (ra != rb) {
        if (ra < rb) {
            int t = ra;
            ra = rb;
            rb = t;
        }
        // hook root ra (larger id) under rb
        unsigned short old = atomicCAS((unsigned short *)&par[ra], (unsigned short)ra,
                                       (unsigned short)rb);
        if (old == ra) return 1;
        ra = old;
    }
    return 0;
}

// Two rows per lane (G64): the lane's rows (2l, 2l+1) form a strip whose run
// overlap graph is a forest (two runs of one row never overlap, so a cycle
// would need two runs of the other row sharing a column). Its components are
// therefore counted without union-find: their spans are disjoint intervals and
// a run start begins a new component unless the other row is set there (ties
// go to the top row): K marks the component starts, popc(K) counts them, and
// the component holding column c is popc(K & (bits <= c)) - 1. Only contacts
// between strips (row 2l vs row 2l-1) go through the shared-memory
// union-find, over strip-component nodes (id = lane * 64 + index).
template <class G>
__device__ __forceinline__ int count_regions_strips(const Team<G> &t, const Bd<G> &pass, uint16_t *par_smem) {
    using Row = typename G::Row;
    volatile uint16_t *par = par_smem;
    const Row A = pass.r[0], Bv = pass.r[1];
    const Row sA = A & ~(A << 1), sB = Bv & ~(Bv << 1);
    const Row K = (sA & (~Bv | sB)) | (sB & ~A);
    const int nk = popc(K);
    const int base = t.lane * G::BITS;
    LG_DCHECK(base + nk <= G::TEAM * G::BITS);
    for (int i = 0; i < nk; i++) par[base + i] = (uint16_t)(base + i);
    const Row Kup = t.up(K), Bup = t.up(Bv);  // lane l-1: strip starts, row 2l-1
    t.sync();
    int links = 0;
    Row C = A & Bup;
    Row CS = C & ~(C << 1);
    while (CS) {  // one union per contact run between row 2l-1 and row 2l
        int c = ctz(CS);
        CS &= CS - 1;
        Row upto = (c == G::BITS - 1) ? ~Row(0) : ((Row(2) << c) - Row(1));
        int i1 = popc(K & upto) - 1, i2 = popc(Kup & upto) - 1;
        LG_DCHECK(t.lane > 0 && i1 >= 0 && i1 < nk && i2 >= 0 && i2 < G::BITS);
        links += uf_unite(par, base + i1, base - G::BITS + i2);
    }
    return t.sum(nk - links);
}

template <class G>
__device__ __forceinline__ int count_regions(const Team<G> &t, const Bd<G> &pass, uint16_t *par_smem) {
    using Row = typename G::Row;
    if constexpr (G::RPL == 2) return count_regions_strips(t, pass, par_smem);
    volatile uint16_t *par = par_smem;
    int runs = 0;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        Row s = pass.r[k] & ~(pass.r[k] << 1);
        int base = t.row(k) * G::RUNS;
        int i = 0;
        while (s) {
            LG_DCHECK(i < G::RUNS);
            par[base + i] = (uint16_t)(base + i);
            i++;
            s &= s - 1;
        }
        runs += i;
    }
    t.sync();
    Row above[G::RPL];
    if constexpr (G::RPL == 1) {
        above[0] = t.up(pass.r[0]);
    } else {
        above[0] = t.up(pass.r[1]);
        above[1] = pass.r[0];
    }
    int links = 0;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int row = t.row(k);
        Row R = pass.r[k], A = above[k];
        Row C = R & A;
        if (row == 0 || C == 0) continue;
        Row SR = R & ~(R << 1), SA = A & ~(A << 1);
        Row CS = C & ~(C << 1);
        while (CS) {
            int c = ctz(CS);
            CS &= CS - 1;
            Row upto = (c == G::BITS - 1) ? ~Row(0) : ((Row(2) << c) - Row(1));
            int ir = popc(SR & upto) - 1, ia = popc(SA & upto) - 1;
            LG_DCHECK(ir >= 0 && ir < G::RUNS && ia >= 0 && ia < G::RUNS && row < G::ROWS);
            links += uf_unite(par, row * G::RUNS + ir, (row - 1) * G::RUNS + ia);
        }
    }
    return t.sum(runs - links);
}

}  // namespace lg
