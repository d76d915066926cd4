// env_kernels.cuh -- the fused batched env step for sm_100a.
//
// One launch of env_kernel<G, DOM> advances a block of E = blockDim/TEAM
// environments (reference _Core.step, levelgen/env.py:355-393) and then
// streams their observations (build_observation, env.py:186-233) to HBM:
//
//   phase 1 (team per env, registers + shared memory)
//     load state -> apply action (narrow/turtle/wide) -> recompute metrics on
//     a real change (problems.py:105-243) -> loss delta reward (251-279) ->
//     advance scan position -> done / info -> in-kernel auto-reset
//     (reset_rows, env.py:284-305, numpy-exact draws) -> store state ->
//     render the env's 0/1 observation planes as a bit image in shared memory
//   phase 2 (same team, no block barrier)
//     expand the env's bit image to float32 with 128-bit streaming stores.
// This lane-team kernel serves maps larger than 16x16 (up to 64x64); smaller
// maps run one env per thread (solo_kernel.cuh).
//
// The observation write is the HBM roofline of the path (15,376 B per env-step
// for binary 16x16 / obs 31 against ~330 B of state traffic).
#pragma once
#include <stdint.h>

#include "rng.cuh"
#include "team.cuh"

namespace lg {

// MODE_RECOMPUTE: metrics + loss after a designer edit (env.py:684-715);
// MODE_REPRICE: loss only, after a target change (env.py:670-681).
enum { MODE_STEP = 0, MODE_RESET = 1, MODE_OBSERVE = 2, MODE_RECOMPUTE = 3, MODE_REPRICE = 4 };
enum { REP_NARROW = 0, REP_TURTLE = 1, REP_WIDE = 2 };
enum { FLAG_BAD_ACTION = 1, FLAG_NO_EDITABLE = 2, FLAG_PINPOINTS = 4 };

// Domain tables (tiles.py:126-171). Stored bit-planes are tile ids 1..N-1
// (plane p <-> tile p+1); AIR is "active and in no plane", BORDER is "inactive".
template <int DOM>
struct Dom;
template <>
struct Dom<0> {  // binary: AIR 0, WALL 1
    static constexpr int N = 2, M = 2, NPL = 1;
};
template <>
struct Dom<1> {  // maze: AIR 0, WALL 1, PLAYER 2, DOOR 3
    static constexpr int N = 4, M = 4, NPL = 3;
};
template <>
struct Dom<2> {  // dungeon: AIR 0, WALL 1, ENEMY 2, KEY 3, DOOR 4, PLAYER 5
    static constexpr int N = 6, M = 7, NPL = 5;
};

struct FastDiv {  // n / d for n, d < 2^31 (mul-hi + shift)
    uint32_t d, mul, shr;
};
__device__ __forceinline__ uint32_t fdiv(const FastDiv &f, uint32_t n) {
    return f.d == 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

// Per-env hot scalars, 32 bytes.
struct __align__(16) Hot {
    uint32_t geo;     // h | w << 8 | pos_r << 16 | pos_c << 24
    int32_t pos_idx;  // narrow scan index
    int32_t order_len;
    int32_t changes;
    int64_t t;
    int64_t max_steps;
};

struct Params {
    // config
    int B, H, W, rep, OH, OW, half;
    int randomize, weighted, n_pins, n_ctrl, det;
    long long max_steps, budget;
    long long n_actions, goffset;
    int pins[16];
    int ctrl[8];
    double cdf[8];
    double w[8];
    // state (library owned)
    void *rows;          // Row [B][NPL+1][ROWS]; plane NPL = frozen
    Hot *hot;            // [B]
    int *mv;             // [B][24]: values 0..6, unreach mask at 7, lo 8..14, hi 16..22
    double *lossv;       // [B][4]: prev_loss, ep_reward, ep_start_loss, -
    ulonglong2 *rs;      // [B][2] PCG state (hi, lo), then (has_uint32 | uinteger << 32, 0):
                         // one 32-byte sector per env, rewritten whole (no partial-sector fill)
    ulonglong2 *ri;      // [B] PCG inc (hi, lo)
    uint2 *rb;           // unused (kept for the layout of Params)
    long long *mseed;    // [B]
    unsigned *err;       // error flags
    // io
    const long long *actions;
    float *obs;
    double *reward;
    unsigned char *done, *terminal;
    double *ep_rew;
    long long *ep_len;
    double *ep_start, *fin_loss;
    double *stats;  // [5]
    const unsigned char *reset_mask;
    // observation writer
    uint32_t PE, PB, OO;  // floats per env, bit-plane elements per env, OH*OW
    FastDiv divPE, divOO;
    int img_words;  // u32 words of one env's bit image (incl. 1 pad word)
    int env_smem;   // shared memory per env: bytes (team kernel) or 32-bit words (solo)
    int solo_E;     // solo kernel: envs per block (== blockDim: warp mode)
    int no_auto_reset;  // scalar step (env.py:611-630): finished envs are not reset
    int obs_u8;         // observation format: 0 = float32 (reference), 1 = uint8 0/1 planes
    int obs_bits;       // packed transfer: `obs` is the batch's 0/1 planes as one u32 bit stream
    int stream_mode;   // solo: envs of a warp/block rendered into one contiguous bit stream
    int group_words;   // solo stream mode: shared words per warp (warp mode) or block
    int stream_words;  // solo stream mode: offset of the union-find scratch in a group
    int off_ctrl;   // byte offset of the control floats within an env's smem
    int off_uf;     // team kernel: byte offset of the union-find scratch within an env's smem
    // solo slot layout: 1 = the frozen plane is not staged because it equals the
    // border plane in every env (no active frozen cell); the writer reads the
    // border plane twice. Decided per launch by the host (lg_env::plain).
    int elide;
    int frz_derived;  // solo: frozen plane == max grid minus episode rect in every env (not read)
    unsigned *aux;  // [1] device flag: an imported env has an active frozen cell
    int early;      // solo warp mode: render + store half the outputs before the recompute
    int coop;       // solo block mode: the warp renders its envs' images together
    int gate;       // validated step (LG_STEP_VALIDATE): skip the launch when the action
                    // check kernel flagged an out-of-range action (no mutation, env.py:358-361)
    // lg_step_random: each env's action is drawn in the step kernel (the draw
    // of lg_random_actions), optionally recorded in act_out
    int rand_act;
    unsigned long long act_seed;
    long long *act_out;
    // chained launches (lg_step_random): per-block tickets [started | done],
    // one pair per block of the launch grid (see chain_enter)
    int chain;
    unsigned *tickets;
};

// Uniform actions: a counter-based draw per (seed, global env index), the
// same values lg_random_actions writes (harness.uniform_policy's role,
// harness.py:149-175, for the device bench loop).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ long long uniform_action(unsigned long long seed, long long gidx, long long n) {
    const uint64_t x = splitmix64(seed * 0xD1B54A32D192ED03ULL ^ splitmix64((uint64_t)gidx));
    return (long long)(((unsigned __int128)x * (unsigned long long)n) >> 64);
}
// the step's action for `env` (record: this thread writes act_out). kRand =
// false compiles the in-kernel draw out (the 64-row lane teams: the host
// draws their actions with random_actions_kernel; see run_mode).
template <bool kRand = true>
__device__ __forceinline__ long long step_action(const Params &p, long long env, bool record) {
    if (kRand && p.rand_act) {
        const long long a = uniform_action(p.act_seed, p.goffset + env, p.n_actions);
        if (record && p.act_out) p.act_out[env] = a;
        return a;
    }
    return p.actions[env];
}

// Episode counters (lg_step's `stats`): finished episodes add into five
// block-shared doubles, flushed to the global counters once per block. A
// lockstep reset step (every env of the batch finishes at once) would
// otherwise send 5 x B double atomics to the same five addresses.
__device__ __forceinline__ double *block_stats() {
    __shared__ double s[5];
    return s;
}
__device__ __forceinline__ bool block_stats_on(const Params &p, int mode) { return p.stats && mode == MODE_STEP; }
__device__ __forceinline__ void block_stats_begin(const Params &p, int mode) {
    if (!block_stats_on(p, mode)) return;
    if (threadIdx.x < 5) block_stats()[threadIdx.x] = 0.0;
    __syncthreads();
}
__device__ __forceinline__ void block_stats_add(double ep_reward, double t, double start, double fin) {
    double *s = block_stats();
    atomicAdd(s + 0, 1.0);
    atomicAdd(s + 1, ep_reward);
    atomicAdd(s + 2, t);
    atomicAdd(s + 3, start);
    atomicAdd(s + 4, fin);
}
__device__ __forceinline__ void block_stats_flush(const Params &p, int mode) {
    if (!block_stats_on(p, mode)) return;
    __syncthreads();
    const double *s = block_stats();
    if (threadIdx.x < 5 && s[0] != 0.0) atomicAdd(p.stats + threadIdx.x, s[threadIdx.x]);
}

// Chained launches. Consecutive lg_step_random launches of one env on one
// stream are programmatic dependent launches: launch k+1 may start while
// launch k's last wave runs. Block j of every launch steps the same envs, so
// it waits only for block j of the previous launch (ticket = the launch's
// sequence number for this block; done[j] counts finished launches), then
// lets the next launch be scheduled. Launch k+1 is only scheduled once every
// block of launch k has passed its wait, so all blocks a waiting block
// depends on are already resident (no deadlock); a wait that does not end
// within 2 s traps (error, not a hang).
__device__ __forceinline__ void chain_enter(const Params &p) {
    if (!p.chain) return;
    if (threadIdx.x == 0) {
        unsigned *started = p.tickets, *done = p.tickets + gridDim.x;
        const unsigned my = atomicAdd(started + blockIdx.x, 1u);
        unsigned v, spins = 0;
        unsigned long long t0 = 0;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + blockIdx.x) : "memory");
            if (v == my) break;
            __nanosleep(128);
            if ((++spins & 1023u) == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (!t0) t0 = now;
                else if (now - t0 > 2000000000ull) __trap();
            }
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void chain_leave(const Params &p) {
    if (!p.chain) return;
    // the barrier orders every thread's stores before thread 0's release (the
    // semaphore pattern: bar.sync, then one st/red.release.gpu; the reader's
    // ld.acquire.gpu, then bar.sync)
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.tickets + gridDim.x + blockIdx.x) : "memory");
}

// Validated steps: the reference rejects a bad action batch before mutating
// anything (env.py:358-361). check_actions_kernel runs first on the stream;
// every thread of the step kernel then reads the same flag word and the whole
// launch returns before touching state.
__device__ __forceinline__ bool gate_closed(const Params &p) {
    return p.gate && (*reinterpret_cast<volatile const unsigned *>(p.err) & FLAG_BAD_ACTION);
}

// Specialised launches. S = 0: every EnvConfig (runtime flags). Otherwise
// S & 3 = 1 + representation, with no controllable metrics, no deterministic
// metrics and float32 observations; S & SPEC_NOPINS also fixes "no pinpoints"
// (the BASELINE configs c1..c5 are all specialised). The flags become
// compile-time constants, so the dead paths leave the kernel: a smaller
// instruction footprint and fewer branches (c4 13.9k -> 9.8k SASS
// instructions, 89 -> 99 M env-steps/s; c2 123 -> 132 M).
constexpr int SPEC_NOPINS = 4;
constexpr int spec_of(int rep, bool nopins) { return 1 + rep + (nopins ? SPEC_NOPINS : 0); }
template <int S> __device__ __forceinline__ int rep_of(const Params &p) { return (S & 3) ? (S & 3) - 1 : p.rep; }
template <int S> __device__ __forceinline__ int nctrl_of(const Params &p) { return (S & 3) ? 0 : p.n_ctrl; }
template <int S> __device__ __forceinline__ int npins_of(const Params &p) { return (S & SPEC_NOPINS) ? 0 : p.n_pins; }
template <int S> __device__ __forceinline__ int det_of(const Params &p) { return (S & 3) ? 0 : p.det; }
template <int S> __device__ __forceinline__ int obs_u8_of(const Params &p) { return (S & 3) ? 0 : p.obs_u8; }
template <int S> __device__ __forceinline__ int obs_bits_of(const Params &p) { return (S & 3) ? 0 : p.obs_bits; }

__device__ __forceinline__ void rng_load(const Params &p, long long env, Pcg &g) {
    const ulonglong2 s = p.rs[2 * env], b = p.rs[2 * env + 1], inc = p.ri[env];
    g.s = ((u128)s.x << 64) | s.y;
    g.inc = ((u128)inc.x << 64) | inc.y;
    g.has = (uint32_t)b.x;
    g.u = (uint32_t)(b.x >> 32);
}
__device__ __forceinline__ void rng_store(const Params &p, long long env, const Pcg &g) {
    p.rs[2 * env] = make_ulonglong2((unsigned long long)(g.s >> 64), (unsigned long long)g.s);
    p.rs[2 * env + 1] = make_ulonglong2((unsigned long long)g.has | ((unsigned long long)g.u << 32), 0ull);
}

template <class G, int DOM>
struct EnvRegs {
    using Row = typename G::Row;
    Bd<G> pl[Dom<DOM>::NPL];  // tile planes
    Bd<G> frz;                // frozen plane
    int h, w, pr, pc, pos_idx, order_len, changes;
    long long t, max_steps;
    int val[8], lo[8], hi[8];
    int unr;
    double prev_loss, ep_reward, ep_start_loss;
    Pcg g;
    long long mseed;
};

template <class G>
__device__ __forceinline__ Bd<G> rect_board(const Team<G> &t, int h, int w) {
    Bd<G> a;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) a.r[k] = t.row(k) < h ? low_mask<typename G::Row>(w) : 0;
    return a;
}

// ---------------------------------------------------------------------------
// metrics (problems.py:105-243) -- values, unreachable mask
// ---------------------------------------------------------------------------

template <class G>
__device__ __forceinline__ int kth_cell(const Team<G> &t, const Bd<G> &m, int k) {
    // flat index (row * 64 + col) of the k-th set cell in row-major order
    int c = m.count();
    int inc = t.scan(c);
    int exc = inc - c;
    unsigned own = t.ballot(exc <= k && k < inc);
    int src = __ffs((int)own) - 1;
    int res = 0;
    if (t.lane == src) {
        int kk = k - exc;
#pragma unroll
        for (int j = 0; j < G::RPL; j++) {
            int cj = popc(m.r[j]);
            if (kk >= 0 && kk < cj) {
                auto x = m.r[j];
                for (int i = 0; i < kk; i++) x &= x - 1;
                res = t.row(j) * 64 + ctz(x);
            }
            kk -= cj;
        }
    }
    return t.from(res, src);
}

template <class G>
__device__ __forceinline__ int lowest_cell(const Team<G> &t, const Bd<G> &m) {
    unsigned own = t.ballot(m.nz());
    int src = __ffs((int)own) - 1;
    int res = 0;
    if (t.lane == src) {
        bool found = false;
#pragma unroll
        for (int j = 0; j < G::RPL; j++)
            if (!found && m.r[j]) {
                res = t.row(j) * 64 + ctz(m.r[j]);
                found = true;
            }
    }
    return t.from(res, src);
}

template <class G>
__device__ __forceinline__ Bd<G> cell_board(const Team<G> &t, int flat) {
    Bd<G> b;
#pragma unroll
    for (int k = 0; k < G::RPL; k++)
        b.r[k] = t.row(k) == (flat >> 6) ? (typename G::Row(1) << (flat & 63)) : 0;
    return b;
}

template <class G>
__device__ __forceinline__ int team_count(const Team<G> &t, const Bd<G> &b) {
    return t.sum(b.count());
}

// Number of distinct connected components of `pass` among the cells of `rem`
// (4-connected): BFS from the lowest remaining cell until every remaining cell
// is reached or the component is exhausted, drop what it reached, repeat.
template <class G>
__device__ __forceinline__ int components_among(const Team<G> &t, Bd<G> rem, const Bd<G> &pass,
                                                typename G::Row wm) {
    int k = 0;
    while (t.any(rem.nz())) {
        ++k;
        Bd<G> f = cell_board(t, lowest_cell(t, rem));
        Bd<G> vis = f;
        while (t.any(andnot(rem, vis).nz())) {
            f = andnot(dilate(t, f, wm) & pass, vis);
            if (!t.any(f.nz())) break;
            vis = vis | f;
        }
        rem = andnot(rem, vis);
    }
    return k;
}

// Backend of the generic metric code for a lane team (team.cuh).
template <class G>
struct TeamK {
    using B = Bd<G>;
    Team<G> t;
    typename G::Row wm;
    __device__ __forceinline__ int count(const B &b) const { return t.sum(b.count()); }
    __device__ __forceinline__ B cell(int flat) const { return cell_board(t, flat); }
    __device__ __forceinline__ int kth(const B &b, int k) const { return kth_cell(t, b, k); }
    __device__ __forceinline__ int lowest(const B &b) const { return lowest_cell(t, b); }
    __device__ __forceinline__ int bfs_last(B &f, const B &pass) const {
        return bfs_last_layer(t, f, pass, wm);
    }
    template <bool ENDPOINT>
    __device__ __forceinline__ void touch(B f, const B &pass, const B &ta, const B &tb, bool want_b,
                                          int &da, int &db) const {
        bfs_touch<G, ENDPOINT>(t, f, pass, wm, ta, tb, want_b, da, db);
    }
    __device__ __forceinline__ int regions(const B &pass, void *uf) const {
        return count_regions(t, pass, reinterpret_cast<uint16_t *>(uf));
    }
    // Change of the region count (count_regions, pathfind.py:116-130) when cell
    // x = (xr, xc) switched passability and nothing else changed: with G the
    // passable set without x and k the number of components of G among x's
    // passable neighbours, adding x merges them into one (1 - k), removing x
    // splits its component into k (k - 1). Exact, and a few BFS layers on
    // typical maps instead of a union-find over the whole grid.
    static constexpr bool kIncRegions = true;
    __device__ __forceinline__ int regions_delta(const B &pass_new, int xr, int xc, bool old_in) const {
        const B x = cell_board(t, xr * 64 + xc);
        const bool new_in = t.any((x & pass_new).nz());
        if (new_in == old_in) return 0;
        const B g = andnot(pass_new, x);
        const int k = components_among(t, dilate(t, x, wm) & g, g, wm);
        return new_in ? 1 - k : k - 1;
    }
};

// compute_metrics_batch for one level (problems.py:105-243), generic over the
// board backend K (lane team or single thread). pl: stored tile planes
// (tile p+1), act: active mask, g: metric generator (binary draw only).
// Incremental region count after a one-cell write (the lane-team kernels'
// steps): the write position, whether the old tile was passable for the
// region metric, and the (exact) count before the write.
struct RegInc {
    int xr, xc;
    bool old_in;
    int old_regions;
};

template <class K, class B>
__device__ __forceinline__ int regions_of(const K &k, const B &pass, void *uf, const RegInc *inc) {
    if constexpr (K::kIncRegions) {
        if (inc) return inc->old_regions + k.regions_delta(pass, inc->xr, inc->xc, inc->old_in);
    }
    return k.regions(pass, uf);
}

template <class K, int DOM>
__device__ __forceinline__ void compute_metrics(const K &k, const typename K::B *pl, const typename K::B &act, Pcg &g,
                                void *uf, int *val, int &unr, const RegInc *inc = nullptr) {
    using B = typename K::B;
    unr = 0;
    if constexpr (DOM == 0) {
        // _binary_metrics (problems.py:136-173)
        B pass = andnot(act, pl[0]);
        val[1] = regions_of(k, pass, uf, inc);
        int cnt = k.count(pass);
        val[0] = 0;
        if (cnt > 0) {
            int kk = (int)pcg_integers(g, 0, cnt);  // problems.py:152-154
            B f = k.cell(k.kth(pass, kk));
            k.bfs_last(f, pass);
            int y = k.lowest(f);  // np.argmax: lowest flat index at max d1
            B f2 = k.cell(y);
            val[0] = k.bfs_last(f2, pass);
        }
    } else if constexpr (DOM == 1) {
        // _maze_metrics (problems.py:176-198): passable AIR | PLAYER | DOOR
        B pass = andnot(act, pl[0]);
        const B &players = pl[1], &doors = pl[2];
        int np = k.count(players), nd = k.count(doors);
        val[2] = np;
        val[3] = nd;
        val[1] = regions_of(k, pass, uf, inc);
        int d = -1, dummy;
        if (np > 0 && nd > 0) k.template touch<false>(players, pass, doors, doors, false, d, dummy);
        bool bad = d < 0;
        val[0] = bad ? 0 : d;
        unr = bad ? 1 : 0;
    } else {
        // _dungeon_metrics (problems.py:201-243); planes WALL ENEMY KEY DOOR PLAYER
        const B &enemy = pl[1], &key = pl[2], &door = pl[3], &player = pl[4];
        B trav = andnot(andnot(andnot(andnot(act, pl[0]), enemy), key), door);  // AIR | PLAYER
        int cp = k.count(player), ck = k.count(key), cd = k.count(door), ce = k.count(enemy);
        val[2] = cp;
        val[3] = ck;
        val[4] = cd;
        val[5] = ce;
        int leg1 = -1, nearv = -1, leg2 = -1, dummy;
        if (cp > 0) k.template touch<true>(player, trav, key, enemy, true, leg1, nearv);
        bool missing = cp == 0 || ck == 0 || cd == 0;
        if (!missing && leg1 >= 0) k.template touch<true>(key, trav, door, door, false, leg2, dummy);
        bool bad = missing || leg1 < 0 || leg2 < 0;
        val[0] = bad ? 0 : leg1 + leg2;
        bool badn = cp == 0 || ce == 0 || nearv < 0;
        val[6] = badn ? 0 : nearv;
        unr = (bad ? 1 : 0) | (badn ? 64 : 0);
        B open = andnot(andnot(act, pl[0]), enemy);  // AIR | PLAYER | KEY | DOOR
        val[1] = regions_of(k, open, uf, inc);
    }
}

// loss_batch (problems.py:251-279): canonical order, explicit IEEE ops (no FMA).
template <int DOM>
__device__ __forceinline__ double loss_of(const Params &p, const int *val, int unr, const int *lo, const int *hi) {
    constexpr int M = Dom<DOM>::M;
    double wreg = p.w[1];
    double total = 0.0;
#pragma unroll
    for (int m = 0; m < M; m++) {
        double wm = p.w[m];
        double x = (double)val[m], l = (double)lo[m], h = (double)hi[m];
        double a = __dsub_rn(l, x), b = __dsub_rn(x, h);
        a = a > 0.0 ? a : 0.0;
        b = b > 0.0 ? b : 0.0;
        double term = __dmul_rn(wm, __dadd_rn(a, b));
        bool path = (DOM == 1 && m == 0) || (DOM == 2 && (m == 0 || m == 6));
        if (path && ((unr >> m) & 1)) term = __dadd_rn(__dmul_rn(wm, h), wreg);
        total = m == 0 ? term : __dadd_rn(total, term);
    }
    return total;
}

// _recompute (env.py:332-347)
// unr bit: the stored region count is exact for the stored map (set by every
// recompute, clear after a state import), so a step may update it incrementally
constexpr int UNR_REGIONS_EXACT = 1 << 15;

// passable for the region metric: binary AIR; maze all but WALL; dungeon all but WALL and ENEMY
template <int DOM>
__device__ __forceinline__ bool regions_pass_tile(int tile) {
    return DOM == 0 ? tile == 0 : DOM == 1 ? tile != 1 : (tile != 1 && tile != 2);
}

template <class G, int DOM, int S = 0>
__device__ __forceinline__ void recompute(const Params &p, const Team<G> &t, EnvRegs<G, DOM> &e, uint16_t *uf,
                          bool reset, const RegInc *inc = nullptr) {
    using Row = typename G::Row;
    TeamK<G> k{t, low_mask<Row>(p.W)};
    Bd<G> act = rect_board(t, e.h, e.w);
    // _metric_rngs (env.py:327-330): the env stream, or a fresh default_rng(metric_seed)
    Pcg mg = e.g;
    if (det_of<S>(p)) seedseq_pcg((uint64_t)e.mseed, false, 0, mg);
    compute_metrics<TeamK<G>, DOM>(k, e.pl, act, mg, uf, e.val, e.unr, inc);
    e.unr |= UNR_REGIONS_EXACT;
    if (!det_of<S>(p)) e.g = mg;
    double l = loss_of<DOM>(p, e.val, e.unr, e.lo, e.hi);
    e.prev_loss = l;
    if (reset) {
        e.ep_reward = 0.0;
        e.ep_start_loss = l;
    }
}

// ---------------------------------------------------------------------------
// scan order (env.py:155-178) without materialising the order array
// ---------------------------------------------------------------------------

// first editable cell in boustrophedon order from row `r0` on (inclusive);
// returns flat row*64+col or -1.
template <class G>
__device__ __forceinline__ int serp_first_from(const Team<G> &t, const Bd<G> &ed, int r0) {
    int best = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int r = t.row(k);
        if (r >= r0 && ed.r[k]) best = min(best, r);
    }
    // team min over rows
    unsigned own = t.ballot(best != 0x7fffffff);
    if (!own) return -1;
    int cand = best;
#pragma unroll
    for (int o = G::TEAM / 2; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(t.mask, cand, o, G::TEAM));
    int row = cand;
    int src = row / G::RPL;
    int res = 0;
    if (t.lane == src) {
#pragma unroll
        for (int k = 0; k < G::RPL; k++)
            if (t.row(k) == row) res = row * 64 + ((row & 1) ? msb(ed.r[k]) : ctz(ed.r[k]));
    }
    return t.from(res, src);
}

// next editable cell strictly after (r, c) in scan order; -1 if none.
template <class G>
__device__ __forceinline__ int serp_next(const Team<G> &t, const Bd<G> &ed, int r, int c) {
    using Row = typename G::Row;
    int src = r / G::RPL;
    int res = -1;
    if (t.lane == src) {
#pragma unroll
        for (int k = 0; k < G::RPL; k++)
            if (t.row(k) == r) {
                Row x = ed.r[k];
                if (r & 1) {
                    Row below = c == 0 ? Row(0) : low_mask<Row>(c);
                    x &= below;
                    if (x) res = r * 64 + msb(x);
                } else {
                    Row above = c >= G::BITS - 1 ? Row(0) : ~low_mask<Row>(c + 1);
                    x &= above;
                    if (x) res = r * 64 + ctz(x);
                }
            }
    }
    res = t.from(res, src);
    if (res >= 0) return res;
    return serp_first_from(t, ed, r + 1);
}

// ---------------------------------------------------------------------------
// reset_rows for one env (env.py:284-325; grid.py:116-225; problems.py:48-90)
// ---------------------------------------------------------------------------

template <class G, int DOM, int S = 0>
__device__ __forceinline__ void reset_env(const Params &p, const Team<G> &t, EnvRegs<G, DOM> &e) {
    using Row = typename G::Row;
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    Pcg &g = e.g;
    int h = p.H, w = p.W;
    if (p.randomize) {  // sample_shape: width then height (grid.py:124-125)
        w = (int)pcg_integers(g, 3, p.W + 1);
        h = (int)pcg_integers(g, 3, p.H + 1);
    }
    e.h = h;
    e.w = w;
    Bd<G> act = rect_board(t, h, w);
#pragma unroll
    for (int q = 0; q < NPL; q++) e.pl[q] = Bd<G>::zero();
    e.frz = andnot(rect_board(t, p.H, p.W), act);  // apply_shape: inactive cells frozen
    if (p.weighted) {
        // init_random: one choice(n_tiles, (h, w), p) block, row-major doubles
        // (grid.py:169-191); each row-lane jumps to its slice of the stream.
#pragma unroll
        for (int k = 0; k < G::RPL; k++) {
            int r = t.row(k);
            if (r < h) {
                Pcg g2 = g;
                pcg_advance(g2, (uint64_t)r * (uint64_t)w);
                for (int c = 0; c < w; c++) {
                    double u = pcg_double(g2);
                    int idx = 0;
#pragma unroll
                    for (int q = 0; q < N; q++) idx += (p.cdf[q] <= u) ? 1 : 0;  // searchsorted right
                    idx = idx < N - 1 ? idx : N - 1;
#pragma unroll
                    for (int q = 0; q < NPL; q++) e.pl[q].r[k] |= (q == idx - 1) ? (Row(1) << c) : Row(0);
                }
            }
        }
        pcg_advance(g, (uint64_t)h * (uint64_t)w);
    }
    if (npins_of<S>(p) > 0) {
        // place_pinpoints: choice(h*w, k, replace=False) over the free cells,
        // which are exactly the h x w rectangle in row-major order here.
        int pop = h * w;
        if (pop < p.n_pins) {
            if (t.lane == 0) atomicOr(p.err, (unsigned)FLAG_PINPOINTS);
        } else {
            int picks[16];
            int k = p.n_pins;
            for (int j = pop - k; j < pop; j++) {  // Floyd
                int val = (int)pcg_bounded(g, (uint64_t)j);
                bool seen = false;
                for (int i = 0; i < j - (pop - k); i++) seen |= picks[i] == val;
                picks[j - (pop - k)] = seen ? j : val;
            }
            for (int i = k - 1; i > 0; i--) {  // bounded Fisher-Yates
                int j = (int)pcg_bounded(g, (uint64_t)i);
                int tmp = picks[i];
                picks[i] = picks[j];
                picks[j] = tmp;
            }
            for (int i = 0; i < k; i++) {
                int r = picks[i] / w, c = picks[i] % w, tile = p.pins[i];
#pragma unroll
                for (int kk = 0; kk < G::RPL; kk++) {
                    const Row m = (t.row(kk) == r) ? (Row(1) << c) : Row(0);
#pragma unroll
                    for (int q = 0; q < NPL; q++)
                        e.pl[q].r[kk] = (e.pl[q].r[kk] & ~m) | (q == tile - 1 ? m : Row(0));
                    e.frz.r[kk] |= m;
                }
            }
        }
    }
    // default_targets + sample_control_targets (problems.py:48-90)
    int cap = h * w;
#pragma unroll
    for (int m = 0; m < M; m++) {
        int lo = 1, hi = 1;
        if (m == 0) lo = hi = cap;  // maximize: diameter / path_length / pkd_path
        if (DOM == 2 && m == 5) {
            lo = 2;
            hi = 5;
        }
        if (DOM == 2 && m == 6) {
            lo = 4;
            hi = cap;
        }
        for (int j = 0; j < nctrl_of<S>(p); j++)
            if (p.ctrl[j] == m) lo = hi = (int)pcg_integers(g, 0, (int64_t)cap + 1);
#pragma unroll
        for (int q = 0; q < 8; q++) {  // select chain keeps the register index static
            e.lo[q] = (q == m) ? lo : e.lo[q];
            e.hi[q] = (q == m) ? hi : e.hi[q];
        }
    }
    if (det_of<S>(p)) e.mseed = (long long)pcg_bounded(g, 0x7FFFFFFFFFFFFFFFULL);  // env.py:302-303
    // _install_row (env.py:307-325)
    Bd<G> ed = andnot(act, e.frz);
    e.order_len = team_count(t, ed);
    int first = serp_first_from(t, ed, 0);
    if (first < 0) {
        if (t.lane == 0) atomicOr(p.err, (unsigned)FLAG_NO_EDITABLE);
        first = 0;
    }
    e.pr = first >> 6;
    e.pc = first & 63;
    e.pos_idx = 0;
    e.t = 0;
    e.changes = 0;
    e.max_steps = p.max_steps > 0 ? p.max_steps : 3LL * cap;
    // the caller runs _recompute(reset=True) (env.py:305)
}

// ---------------------------------------------------------------------------
// state load / store
// ---------------------------------------------------------------------------

template <class G, int DOM>
__device__ __forceinline__ typename G::Row *rows_of(const Params &p, long long env) {
    return reinterpret_cast<typename G::Row *>(p.rows) +
           (size_t)env * (Dom<DOM>::NPL + 1) * G::ROWS;
}

template <class G, int DOM, int S = 0>
__device__ __forceinline__ void load_env(const Params &p, const Team<G> &t, long long env, EnvRegs<G, DOM> &e) {
    constexpr int NPL = Dom<DOM>::NPL;
    const typename G::Row *rw = rows_of<G, DOM>(p, env);
#pragma unroll
    for (int q = 0; q <= NPL; q++) {
#pragma unroll
        for (int k = 0; k < G::RPL; k++) {
            auto v = rw[q * G::ROWS + t.row(k)];
            if (q < NPL) e.pl[q].r[k] = v;
            else e.frz.r[k] = v;
        }
    }
    Hot hv = p.hot[env];
    e.h = hv.geo & 255;
    e.w = (hv.geo >> 8) & 255;
    e.pr = (hv.geo >> 16) & 255;
    e.pc = hv.geo >> 24;
    e.pos_idx = hv.pos_idx;
    e.order_len = hv.order_len;
    e.changes = hv.changes;
    e.t = hv.t;
    e.max_steps = hv.max_steps;
    const int4 *mv = reinterpret_cast<const int4 *>(p.mv + env * 24);
    int4 a = mv[0], b = mv[1], c = mv[2], d = mv[3], f = mv[4], h2 = mv[5];
    e.val[0] = a.x; e.val[1] = a.y; e.val[2] = a.z; e.val[3] = a.w;
    e.val[4] = b.x; e.val[5] = b.y; e.val[6] = b.z; e.unr = b.w;
    e.lo[0] = c.x; e.lo[1] = c.y; e.lo[2] = c.z; e.lo[3] = c.w;
    e.lo[4] = d.x; e.lo[5] = d.y; e.lo[6] = d.z; e.lo[7] = d.w;
    e.hi[0] = f.x; e.hi[1] = f.y; e.hi[2] = f.z; e.hi[3] = f.w;
    e.hi[4] = h2.x; e.hi[5] = h2.y; e.hi[6] = h2.z; e.hi[7] = h2.w;
    const double2 *lv = reinterpret_cast<const double2 *>(p.lossv + env * 4);
    double2 l0 = lv[0], l1 = lv[1];
    e.prev_loss = l0.x;
    e.ep_reward = l0.y;
    e.ep_start_loss = l1.x;
    rng_load(p, env, e.g);
    e.mseed = det_of<S>(p) ? p.mseed[env] : 0;
}

template <class G, int DOM, int S = 0>
__device__ __forceinline__ void store_env(const Params &p, const Team<G> &t, long long env, const EnvRegs<G, DOM> &e,
                          bool rows_dirty, int dirty_row, bool metrics_dirty, bool rng_dirty) {
    constexpr int NPL = Dom<DOM>::NPL;
    if (rows_dirty || dirty_row >= 0) {
        typename G::Row *rw = rows_of<G, DOM>(p, env);
        constexpr int SEC = 32 / (int)sizeof(typename G::Row);  // rows per 32-byte sector
#pragma unroll
        for (int k = 0; k < G::RPL; k++) {
            int r = t.row(k);
            // the whole sector around the edited row (no partial-sector read-fill)
            if (rows_dirty || (dirty_row >= 0 && r / SEC == dirty_row / SEC)) {
#pragma unroll
                for (int q = 0; q < NPL; q++) rw[q * G::ROWS + r] = e.pl[q].r[k];
                if (rows_dirty) rw[NPL * G::ROWS + r] = e.frz.r[k];
            }
        }
    }
    if (t.lane != 0) return;
    Hot hv;
    hv.geo = (uint32_t)e.h | ((uint32_t)e.w << 8) | ((uint32_t)e.pr << 16) | ((uint32_t)e.pc << 24);
    hv.pos_idx = e.pos_idx;
    hv.order_len = e.order_len;
    hv.changes = e.changes;
    hv.t = e.t;
    hv.max_steps = e.max_steps;
    p.hot[env] = hv;
    if (metrics_dirty) {
        int4 *mv = reinterpret_cast<int4 *>(p.mv + env * 24);
        mv[0] = make_int4(e.val[0], e.val[1], e.val[2], e.val[3]);
        mv[1] = make_int4(e.val[4], e.val[5], e.val[6], e.unr);
        mv[2] = make_int4(e.lo[0], e.lo[1], e.lo[2], e.lo[3]);
        mv[3] = make_int4(e.lo[4], e.lo[5], e.lo[6], e.lo[7]);
        mv[4] = make_int4(e.hi[0], e.hi[1], e.hi[2], e.hi[3]);
        mv[5] = make_int4(e.hi[4], e.hi[5], e.hi[6], e.hi[7]);
    }
    double2 *lv = reinterpret_cast<double2 *>(p.lossv + env * 4);
    lv[0] = make_double2(e.prev_loss, e.ep_reward);
    lv[1] = make_double2(e.ep_start_loss, 0.0);
    if (rng_dirty) {
        rng_store(p, env, e.g);
        if (det_of<S>(p)) p.mseed[env] = e.mseed;
    }
}

// ---------------------------------------------------------------------------
// observation bit image (env.py:186-233)
// ---------------------------------------------------------------------------

// OR a row of `nbits` (<=128) window bits into the image at bit offset `off`.
__device__ __forceinline__ void img_or(uint32_t *img, uint32_t off, u128 v) {
    if (v == 0) return;
    uint32_t w0 = off >> 5, sh = off & 31;
    u128 lo = v << sh;
    uint32_t hi = sh ? (uint32_t)(v >> (128 - sh)) : 0u;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t x = (uint32_t)(lo >> (32 * j));
        if (x) atomicOr(&img[w0 + j], x);
    }
    if (hi) atomicOr(&img[w0 + 4], hi);
}

// OR a window row of <= 32 bits into the image at bit offset `off`.
__device__ __forceinline__ void img_or64(uint32_t *img, uint32_t off, uint64_t v) {
    if (v == 0) return;
    uint64_t x = v << (off & 31);
    uint32_t w0 = off >> 5;
    if ((uint32_t)x) atomicOr(&img[w0], (uint32_t)x);
    if ((uint32_t)(x >> 32)) atomicOr(&img[w0 + 1], (uint32_t)(x >> 32));
}

// Column masks of an observation window starting at grid column c0: bits of
// window columns inside the max grid, and all OW bits.
struct WinMask {
    u128 inside, full;
    __device__ __forceinline__ WinMask(int c0, int OW, int W) {
        int jlo = c0 < 0 ? -c0 : 0;
        int jhi = W - c0;
        if (jhi > OW) jhi = OW;
        inside = 0;
        if (jhi > jlo) {
            u128 upto = jhi >= 128 ? ~(u128)0 : (((u128)1 << jhi) - 1);
            inside = upto & ~(((u128)1 << jlo) - 1);
        }
        full = OW >= 128 ? ~(u128)0 : (((u128)1 << OW) - 1);
    }
};

// Window row bits of one grid row word: column c0+j -> bit j; columns
// outside the max grid read `fill`.
__device__ __forceinline__ u128 window_bits(uint64_t gridrow, int c0, const WinMask &m, bool fill) {
    u128 x = (u128)gridrow;
    u128 win = c0 >= 0 ? (x >> c0) : (x << (-c0));
    win &= m.inside;
    if (fill) win |= m.full & ~m.inside;
    return win;
}
// the same for windows of <= 32 columns, in 64-bit arithmetic
__device__ __forceinline__ uint64_t window_bits64(uint64_t gridrow, int c0, uint64_t inside, uint64_t full,
                                                  bool fill) {
    uint64_t win = c0 >= 0 ? (gridrow >> c0) : (gridrow << (-c0));
    win &= inside;
    if (fill) win |= full & ~inside;
    return win;
}

// A/B knobs for the team kernel's code size (instruction-cache pressure on
// 64x64 maps): default keeps the renderer inlined and leaves the writers to nvcc.
#ifndef LG_TEAM_RENDER_ATTR
#define LG_TEAM_RENDER_ATTR __forceinline__
#endif
#ifndef LG_TEAM_WRITER_ATTR
#define LG_TEAM_WRITER_ATTR
#endif

template <class G, int DOM, int S = 0>
__device__ LG_TEAM_RENDER_ATTR void render_env(const Params &p, const Team<G> &t, const EnvRegs<G, DOM> &e,
                           unsigned char *es) {
    using Row = typename G::Row;
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL;
    uint32_t *img = reinterpret_cast<uint32_t *>(es);
    for (int i = t.lane; i < p.img_words; i += G::TEAM) img[i] = 0;
    // control planes: (value - (lo+hi)/2) / cap in float64, stored as float32
    float *ctrl = reinterpret_cast<float *>(es + p.off_ctrl);
    if (t.lane < nctrl_of<S>(p)) {
        int m = p.ctrl[t.lane];
        int vm = 0, lm = 0, hm = 0;
#pragma unroll
        for (int q = 0; q < 8; q++)
            if (q == m) {
                vm = e.val[q];
                lm = e.lo[q];
                hm = e.hi[q];
            }
        double tgt = __ddiv_rn(__dadd_rn((double)lm, (double)hm), 2.0);
        double v = __ddiv_rn(__dsub_rn((double)vm, tgt), (double)(e.h * e.w));
        ctrl[t.lane] = __double2float_rn(v);
    }
    t.sync();
    int r0 = 0, c0 = 0;
    if (rep_of<S>(p) != REP_WIDE) {
        r0 = e.pr - p.half;
        c0 = e.pc - p.half;
    }
    const int OH = p.OH, OW = p.OW;
    const uint32_t plane_bits = (uint32_t)OH * OW;
    Row wmask = low_mask<Row>(p.W);
    const WinMask wm(c0, OW, p.W);
    const bool narrow_win = OW <= 32;  // 64-bit window arithmetic suffices (uniform)
    const uint64_t in64 = (uint64_t)wm.inside, full64 = (uint64_t)wm.full;
    // rows inside the max grid, emitted by the lane that holds them
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int gr = t.row(k);
        int i = gr - r0;
        if (gr < p.H && i >= 0 && i < OH) {
            Row act = gr < e.h ? low_mask<Row>(e.w) : Row(0);
            Row any = 0;
#pragma unroll
            for (int q = 0; q < NPL; q++) any |= e.pl[q].r[k];
            const uint32_t rowoff = (uint32_t)i * OW;
            LG_DCHECK((N + 1) * plane_bits + rowoff + OW <= (uint32_t)p.img_words * 32);
            uint64_t rows[N + 2];
            rows[0] = (uint64_t)(act & ~any);
#pragma unroll
            for (int q = 0; q < NPL; q++) rows[q + 1] = (uint64_t)e.pl[q].r[k];
            rows[N] = (uint64_t)(~act & wmask);
            rows[N + 1] = (uint64_t)e.frz.r[k];
#pragma unroll
            for (int q = 0; q < N + 2; q++) {
                const bool fill = q >= N;  // border and frozen read 1 outside the grid
                if (narrow_win)
                    img_or64(img, q * plane_bits + rowoff, window_bits64(rows[q], c0, in64, full64, fill));
                else
                    img_or(img, q * plane_bits + rowoff, window_bits(rows[q], c0, wm, fill));
            }
        }
    }
    // window rows outside the max grid: border and frozen everywhere
    for (int i = t.lane; i < OH; i += G::TEAM) {
        int gr = r0 + i;
        if (gr < 0 || gr >= p.H) {
            if (narrow_win) {
                img_or64(img, N * plane_bits + (uint32_t)i * OW, full64);
                img_or64(img, (N + 1) * plane_bits + (uint32_t)i * OW, full64);
            } else {
                img_or(img, N * plane_bits + (uint32_t)i * OW, wm.full);
                img_or(img, (N + 1) * plane_bits + (uint32_t)i * OW, wm.full);
            }
        }
    }
}

// Expand one env's bit image to float32: its output range is written by the
// env's own team (no block barrier), with 16-byte streaming stores.
__device__ __forceinline__ float team_elem(const Params &p, const unsigned char *es, uint32_t le) {
    if (le < p.PB) {
        const uint32_t *img = reinterpret_cast<const uint32_t *>(es);
        return ((img[le >> 5] >> (le & 31)) & 1u) ? 1.0f : 0.0f;
    }
    return reinterpret_cast<const float *>(es + p.off_ctrl)[fdiv(p.divOO, le - p.PB)];
}

// 4 bits -> 4 bytes of 0/1 (bit k lands in byte k).
__device__ __forceinline__ uint32_t bits_to_bytes4(uint32_t x) { return ((x & 0xFu) * 0x00204081u) & 0x01010101u; }

// uint8 observation (opt-in, no control planes): 16 elements per 16-byte store.
template <class G>
__device__ LG_TEAM_WRITER_ATTR void write_obs_team_u8(const Params &p, const Team<G> &t, long long env, const unsigned char *es) {
    const uint32_t *img = reinterpret_cast<const uint32_t *>(es);
    const size_t base = (size_t)env * p.PE;
    uint8_t *out = reinterpret_cast<uint8_t *>(p.obs) + base;
    uint32_t head = (uint32_t)((16 - (base & 15)) & 15);
    if (head > p.PE) head = p.PE;
    for (uint32_t e = t.lane; e < head; e += G::TEAM) out[e] = (img[e >> 5] >> (e & 31)) & 1u;
    const uint32_t n16 = (p.PE - head) >> 4;
    uint4 *o16 = reinterpret_cast<uint4 *>(out + head);
    for (uint32_t q = t.lane; q < n16; q += G::TEAM) {
        uint32_t le = head + (q << 4);
        uint32_t x = __funnelshift_r(img[le >> 5], img[(le >> 5) + 1], le & 31);
        __stcs(o16 + q, make_uint4(bits_to_bytes4(x), bits_to_bytes4(x >> 4), bits_to_bytes4(x >> 8),
                                   bits_to_bytes4(x >> 12)));
    }
    for (uint32_t e = head + (n16 << 4) + t.lane; e < p.PE; e += G::TEAM)
        out[e] = (img[e >> 5] >> (e & 31)) & 1u;
}

// Packed transfer (see solo_write_bits): env's PE bits at stream bits
// [env*PE, env*PE + PE); words shared with a neighbouring env are OR-ed into
// the zeroed stream, the ends of the batch are stored.
template <class G>
__device__ LG_TEAM_WRITER_ATTR void write_obs_team_bits(const Params &p, const Team<G> &t, long long env, const unsigned char *es) {
    const uint32_t *img = reinterpret_cast<const uint32_t *>(es);
    uint32_t *out = reinterpret_cast<uint32_t *>(p.obs);
    const uint32_t PE = p.PE;
    const unsigned long long g0 = (unsigned long long)env * PE;
    const uint32_t sh = (uint32_t)(g0 & 31), nw = (sh + PE + 31) >> 5;
    const unsigned long long w0 = g0 >> 5;
    for (uint32_t i = t.lane; i < nw; i += G::TEAM) {
        uint32_t v, lp;  // local bits [lp, lp + 32) land at bits [0, 32) (or [sh, 32) for word 0)
        if (i == 0) {
            v = img[0];
            lp = 0;
        } else {
            lp = 32 * i - sh;
            v = __funnelshift_r(img[lp >> 5], img[(lp >> 5) + 1], lp & 31);
        }
        const uint32_t avail = PE - lp;  // local bits left from lp
        if (avail < 32) v &= (1u << avail) - 1u;
        if (i == 0) v <<= sh;
        const bool shared = (i == 0 && sh && env > 0) || (i == nw - 1 && ((sh + PE) & 31) && env + 1 < p.B);
        if (shared) atomicOr(out + w0 + i, v);
        else out[w0 + i] = v;
    }
}

template <class G>
__device__ LG_TEAM_WRITER_ATTR void write_obs_team(const Params &p, const Team<G> &t, long long env, const unsigned char *es) {
    const uint32_t *img = reinterpret_cast<const uint32_t *>(es);
    const size_t base = (size_t)env * p.PE;
    float *out = p.obs + base;
    uint32_t head = (uint32_t)((4 - (base & 3)) & 3);
    if (head > p.PE) head = p.PE;
    for (uint32_t e = t.lane; e < head; e += G::TEAM) out[e] = team_elem(p, es, e);
    const uint32_t n4 = (p.PE - head) >> 2;
    float4 *o4 = reinterpret_cast<float4 *>(out + head);
    for (uint32_t q = t.lane; q < n4; q += G::TEAM) {
        uint32_t le = head + (q << 2);
        float4 v;
        if (le + 3 < p.PB) {
            uint32_t wi = le >> 5;
            uint32_t x = __funnelshift_r(img[wi], img[wi + 1], le & 31);
            v.x = (x & 1u) ? 1.0f : 0.0f;
            v.y = (x & 2u) ? 1.0f : 0.0f;
            v.z = (x & 4u) ? 1.0f : 0.0f;
            v.w = (x & 8u) ? 1.0f : 0.0f;
        } else {
            v.x = team_elem(p, es, le);
            v.y = team_elem(p, es, le + 1);
            v.z = team_elem(p, es, le + 2);
            v.w = team_elem(p, es, le + 3);
        }
        __stcs(o4 + q, v);
    }
    for (uint32_t e = head + (n4 << 2) + t.lane; e < p.PE; e += G::TEAM) out[e] = team_elem(p, es, e);
}

// The specialised kernels' writer (no control planes: every element is a bit
// of the image): 32-byte streaming stores (st.global.cs.v8.f32), 8 elements
// from one funnel shift, after a head of at most 7 elements up to 32-byte
// alignment (a c2 observation is 23,064 bytes, so env outputs start at any
// multiple of 8 bytes).
__device__ __forceinline__ void team_st_v8(float *ptr, const float *v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// [qa, qb): the 8-element groups to write, in eighths of the env's groups
// (the early path writes part before the recompute, the rest after it); the
// head and tail elements go with the first / last part.
template <class G>
__device__ LG_TEAM_WRITER_ATTR void write_obs_team_nc(const Params &p, const Team<G> &t, long long env, const unsigned char *es,
                                                    int part_lo = 0, int part_hi = 8) {
    const uint32_t *img = reinterpret_cast<const uint32_t *>(es);
    const uint32_t PE = p.PE;
    float *out = p.obs + (size_t)env * PE;
    uint32_t head = (uint32_t)(((32u - (uint32_t)(reinterpret_cast<uintptr_t>(out) & 31u)) & 31u) >> 2);
    if (head > PE) head = PE;
    const uint32_t n8 = (PE - head) >> 3;
    const uint32_t qa = n8 * (uint32_t)part_lo / 8, qb = n8 * (uint32_t)part_hi / 8;
    if (part_lo == 0)
        for (uint32_t e = t.lane; e < head; e += G::TEAM) out[e] = ((img[e >> 5] >> (e & 31)) & 1u) ? 1.0f : 0.0f;
    for (uint32_t q = qa + t.lane; q < qb; q += G::TEAM) {
        const uint32_t le = head + (q << 3), wi = le >> 5;
        const uint32_t x = __funnelshift_r(img[wi], img[wi + 1], le & 31);
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; j++) f[j] = (x & (1u << j)) ? 1.0f : 0.0f;
        team_st_v8(out + le, f);
    }
    if (part_hi == 8)
        for (uint32_t e = head + (n8 << 3) + t.lane; e < PE; e += G::TEAM)
            out[e] = ((img[e >> 5] >> (e & 31)) & 1u) ? 1.0f : 0.0f;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------

#ifndef LG_TEAM_EARLY_SPLIT
#define LG_TEAM_EARLY_SPLIT 1  // eighths of an env's output stored before its recompute (specialised kernels)
#endif
// Chained launches, in-kernel random actions and block-aggregated episode
// counters are compiled into the lane teams of one row per lane only: the
// 64-row kernel (c4) is bound by instruction fetch (the chain code measured
// 277 -> 264 M env-steps/s), and it runs one env per block anyway.
template <class G>
constexpr bool kTeamChain = G::RPL == 1;

template <class G, int DOM, int S = 0>
__device__ __forceinline__ void env_team_body(const Params &p, int mode) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Row = typename G::Row;
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL;
    Team<G> t;
    const int E = blockDim.x / G::TEAM;
    const int ti = threadIdx.x / G::TEAM;
    const long long env = (long long)blockIdx.x * E + ti;
    // the specialised kernels of maps <= 32 rows store part of the observation
    // after the recompute, so their union-find scratch follows the bit image;
    // otherwise it aliases the image (64x64: c4's 7x7 window is written whole
    // before the recompute, the separate scratch measured 5% slower)
    constexpr int kSplit = (S != 0 && G::RPL == 1) ? LG_TEAM_EARLY_SPLIT : 8;
    unsigned char *es = smem + (size_t)ti * p.env_smem;
    uint16_t *uf = reinterpret_cast<uint16_t *>(es + (kSplit < 8 ? p.off_uf : 0));
    if (gate_closed(p)) return;

    if (env < p.B) {
        EnvRegs<G, DOM> e;
        load_env<G, DOM, S>(p, t, env, e);
        bool rows_dirty = false, metrics_dirty = false, rng_dirty = false;
        bool wrote = false, reset_now = false;
        double before = 0.0;
        int dirty_row = -1, wcol = 0, wcur = 0;  // the write (row, column, old tile)
        if (mode == MODE_STEP) {
            long long a = step_action<kTeamChain<G>>(p, env, t.lane == 0);
            bool ok = a >= 0 && a < p.n_actions;
            if (!ok && t.lane == 0) atomicOr(p.err, (unsigned)FLAG_BAD_ACTION);
            int r = e.pr, c = e.pc, tile = -1;
            if (rep_of<S>(p) == REP_NARROW) {
                if (ok && a != 0) tile = (int)a - 1;
            } else if (rep_of<S>(p) == REP_TURTLE) {
                if (ok && a < 4) {  // moves, clamped to the episode rectangle
                    if (a == 0) r = r > 0 ? r - 1 : 0;
                    else if (a == 1) r = r < e.h - 1 ? r + 1 : e.h - 1;
                    else if (a == 2) c = c > 0 ? c - 1 : 0;
                    else c = c < e.w - 1 ? c + 1 : e.w - 1;
                    e.pr = r;
                    e.pc = c;
                } else if (ok) {
                    tile = (int)a - 4;
                }
            } else {  // wide
                if (ok) {
                    long long cell = a / N;
                    tile = (int)(a - cell * N);
                    r = (int)(cell / p.W);
                    c = (int)(cell - (long long)r * p.W);
                }
            }
            // tile currently at (r, c) and editability, from the owning lane
            int cur = 0, editable = 0;
            int src = r / G::RPL;
            if (t.lane == src) {
#pragma unroll
                for (int k = 0; k < G::RPL; k++)
                    if (t.row(k) == r) {
                        Row bit = Row(1) << c;
                        bool act = r < e.h && c < e.w;
                        cur = act ? 0 : N;
#pragma unroll
                        for (int q = 0; q < NPL; q++)
                            if (e.pl[q].r[k] & bit) cur = q + 1;
                        editable = act && !(e.frz.r[k] & bit);
                    }
            }
            cur = t.from(cur, src);
            editable = t.from(editable, src);
            // narrow: the scan cell is always editable (env.py:366-367)
            wrote = tile >= 0 && tile != cur && (rep_of<S>(p) == REP_NARROW || editable);
            if (wrote) {  // env.py:369-372
                // branch-free value selects (no conditional stores into the
                // register-resident planes, which would force them to local memory)
#pragma unroll
                for (int k = 0; k < G::RPL; k++) {
                    const Row m = (t.row(k) == r) ? (Row(1) << c) : Row(0);
#pragma unroll
                    for (int q = 0; q < NPL; q++) e.pl[q].r[k] = (e.pl[q].r[k] & ~m) | (q == tile - 1 ? m : Row(0));
                }
                dirty_row = r;
                wcol = c;
                wcur = cur;
                e.changes += 1;
                before = e.prev_loss;
            }
        } else if (mode == MODE_RESET) {
            reset_now = !p.reset_mask || p.reset_mask[env];
        } else if (mode == MODE_RECOMPUTE) {
            wrote = !p.reset_mask || p.reset_mask[env];  // recompute without a write
        } else if (mode == MODE_REPRICE) {
            if (!p.reset_mask || p.reset_mask[env]) e.prev_loss = loss_of<DOM>(p, e.val, e.unr, e.lo, e.hi);
        }
        bool ends = false, early = false;
        if (mode == MODE_STEP) {
            // scan advance and t (env.py:374-381) do not depend on the recompute
            if (rep_of<S>(p) == REP_NARROW) {  // pos_idx = (pos_idx + 1) % order_len
                int nidx = e.pos_idx + 1;
                int nxt;
                Bd<G> ed = andnot(rect_board(t, e.h, e.w), e.frz);
                if (nidx >= e.order_len) {
                    nidx = 0;
                    nxt = serp_first_from(t, ed, 0);
                } else {
                    nxt = serp_next(t, ed, e.pr, e.pc);
                }
                nxt = max(nxt, 0);  // no editable cell left (imported state): stay well-formed
                e.pos_idx = nidx;
                e.pr = nxt >> 6;
                e.pc = nxt & 63;
            }
            e.t += 1;
            ends = e.t >= e.max_steps || (p.budget > 0 && e.changes >= p.budget);
            // early observation: unless the episode ends (auto-reset) or control
            // planes show metric values, the observation is final now -- write
            // it before the recompute so its stores drain while the team computes
// the specialised 64x64 kernel renders once, after the recompute: with the
// incremental region count its step is short, the 7x7 window is 784 B, and
// the second render/writer copy of the early path costs instruction fetch
// (no_inst was 41% of stalls): c4 250 -> 276 M env-steps/s
#ifndef LG_G64_SPEC_EARLY
#define LG_G64_SPEC_EARLY 0
#endif
            constexpr bool kEarlyOk = S == 0 || G::RPL == 1 || LG_G64_SPEC_EARLY;
            early = kEarlyOk && p.early && p.obs && nctrl_of<S>(p) == 0 && !ends;
            if (early) {
                t.sync();
                render_env<G, DOM, S>(p, t, e, es);
                t.sync();
                if (obs_bits_of<S>(p)) write_obs_team_bits<G>(p, t, env, es);
                else if (obs_u8_of<S>(p)) write_obs_team_u8<G>(p, t, env, es);
                // specialised kernels: part of the output now, the rest after the
                // recompute (no launch-wide phase of computing without storing)
                else if constexpr (S != 0) write_obs_team_nc<G>(p, t, env, es, 0, kSplit);
                else write_obs_team<G>(p, t, env, es);
                if constexpr (kSplit == 8) t.sync();  // the image doubles as union-find scratch
            }
        }
        // pass 0: the step's recompute + bookkeeping; pass 1: auto-reset (one
        // call site for the metric code keeps the instruction footprint small)
#pragma unroll 1
        for (int pass = 0; pass < 2; pass++) {
            if (pass == 1) {
                if (!reset_now) break;
                reset_env<G, DOM, S>(p, t, e);
                rows_dirty = true;
            }
            if (pass == 1 || wrote) {
                // a step's one-cell write updates the region count incrementally
                // (TeamK::regions_delta) when the stored count is exact
                RegInc ri{dirty_row, wcol, regions_pass_tile<DOM>(wcur), e.val[1]};
                const bool inc = pass == 0 && mode == MODE_STEP && (e.unr & UNR_REGIONS_EXACT);
                recompute<G, DOM, S>(p, t, e, uf, pass == 1, inc ? &ri : nullptr);  // _recompute (env.py:332-347)
                metrics_dirty = rng_dirty = true;
            }
            if (pass == 0 && mode == MODE_STEP) {
                double reward = wrote ? __dsub_rn(before, e.prev_loss) : 0.0;
                e.ep_reward = __dadd_rn(e.ep_reward, reward);
                const bool done = ends;
                if (t.lane == 0) {
                    p.reward[env] = reward;
                    p.done[env] = done;
                    if (p.terminal) p.terminal[env] = done;
                    if (p.ep_rew) p.ep_rew[env] = done ? e.ep_reward : 0.0;
                    if (p.ep_len) p.ep_len[env] = done ? e.t : 0;
                    if (p.ep_start) p.ep_start[env] = done ? e.ep_start_loss : 0.0;
                    if (p.fin_loss) p.fin_loss[env] = done ? e.prev_loss : 0.0;
                    if (done && p.stats) {
                        if constexpr (kTeamChain<G>) {
                            block_stats_add(e.ep_reward, (double)e.t, e.ep_start_loss, e.prev_loss);
                        } else {  // 64-row teams: one env per block, the counters directly
                            atomicAdd(p.stats + 0, 1.0);
                            atomicAdd(p.stats + 1, e.ep_reward);
                            atomicAdd(p.stats + 2, (double)e.t);
                            atomicAdd(p.stats + 3, e.ep_start_loss);
                            atomicAdd(p.stats + 4, e.prev_loss);
                        }
                    }
                }
                reset_now = done && !p.no_auto_reset;
            }
        }
        if (mode != MODE_OBSERVE) store_env<G, DOM, S>(p, t, env, e, rows_dirty, dirty_row, metrics_dirty, rng_dirty);
        if (p.obs && !early) {
            t.sync();
            render_env<G, DOM, S>(p, t, e, es);
            t.sync();
            if (obs_bits_of<S>(p)) write_obs_team_bits<G>(p, t, env, es);
            else if (obs_u8_of<S>(p)) write_obs_team_u8<G>(p, t, env, es);
            else if constexpr (S != 0) write_obs_team_nc<G>(p, t, env, es);
            else write_obs_team<G>(p, t, env, es);
        } else if constexpr (S != 0 && kSplit < 8) {
            if (p.obs && early) write_obs_team_nc<G>(p, t, env, es, kSplit, 8);
        }
    }
}

// Residency target per kernel: G::MINB, except the specialised 64-row kernel
// (c4), which runs spill-free at 96 registers (MINB 10: 277 vs 272 M
// env-steps/s at 64 registers with 266 B of spills; its occupancy at 64 was
// capped at 32 one-warp blocks per SM anyway). The generic 64-row kernels
// keep 16 (at 96 registers: 65,536 envs -3%, 4,096 envs +7%).
#ifndef LG_G64_SPEC_MINB
#define LG_G64_SPEC_MINB 10
#endif
template <class G, int S>
constexpr int team_minb() {
    return (S != 0 && G::RPL == 2) ? LG_G64_SPEC_MINB : G::MINB;
}

template <class G, int DOM, int S = 0>
__global__ void __launch_bounds__(64, team_minb<G, S>()) env_kernel(const Params p, int mode) {
    if constexpr (kTeamChain<G>) {
        chain_enter(p);
        block_stats_begin(p, mode);
    }
    env_team_body<G, DOM, S>(p, mode);
    if constexpr (kTeamChain<G>) {
        block_stats_flush(p, mode);
        chain_leave(p);
    }
}

}  // namespace lg
