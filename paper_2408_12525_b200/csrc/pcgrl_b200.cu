// pcgrl_b200.cu -- C ABI (include/pcgrl_b200.h) over the sm_100a env kernels.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <new>
#include <set>
#include <type_traits>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/pcgrl_b200.h"
#include "env_kernels.cuh"
#include "host_expand.h"
#include "policy_kernels.cuh"
#include "solo_kernel.cuh"
#include "trunk_kernel.cuh"

using namespace lg;

static thread_local char g_err[512];
static void set_err(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
extern "C" const char *lg_last_error(void) { return g_err; }
extern "C" const char *lg_version(void) { return "pcgrl_b200 0.1 sm_100a"; }

#define CU(call)                                                           \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) {                                           \
            set_err("CUDA error: %s (line %d)", cudaGetErrorString(_e), __LINE__); \
            return LG_ECUDA;                                               \
        }                                                                  \
    } while (0)

// Switches to the env's device for the duration of a call and restores the
// caller's current device afterwards (a library call must not leave the
// process on another GPU).
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
        else if (err == cudaSuccess) prev = -1;  // already current: nothing to restore
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
#define DEVICE_GUARD(dev)       \
    DeviceGuard _dg(dev);       \
    CU(_dg.err)

// NVTX ranges around every library call that launches work (nsys / ncu
// --nvtx attribute kernels to them; without a tool attached they cost a
// few nanoseconds).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
static const char *mode_name(int mode) {
    switch (mode) {
    case MODE_STEP: return "lg_step";
    case MODE_RESET: return "lg_reset";
    case MODE_OBSERVE: return "lg_observe";
    case MODE_RECOMPUTE: return "lg_recompute";
    default: return "lg_reprice";
    }
}

// The dynamic shared memory limit is a per-device function attribute: raise it
// once per (kernel, device) pair, on the current device.
static cudaError_t smem_attr(const void *fn, int bytes = 200 * 1024) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

// ---------------------------------------------------------------------------
// auxiliary kernels
// ---------------------------------------------------------------------------

__global__ void seed_kernel(long long B, unsigned long long seed, long long offset, ulonglong2 *rs,
                            ulonglong2 *ri, uint2 *rb) {
    long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    Pcg g;
    seedseq_pcg(seed, true, (uint64_t)(offset + b), g);
    rs[2 * b] = make_ulonglong2((unsigned long long)(g.s >> 64), (unsigned long long)g.s);
    rs[2 * b + 1] = make_ulonglong2(0ull, 0ull);  // has_uint32 = 0, uinteger = 0
    ri[b] = make_ulonglong2((unsigned long long)(g.inc >> 64), (unsigned long long)g.inc);
}

__global__ void random_actions_kernel(long long B, long long goffset, unsigned long long seed,
                                      long long n_actions, long long *out) {
    long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    out[b] = uniform_action(seed, goffset + b, n_actions);
}

// Validated steps (env.py:358-361): flags an out-of-range action before the
// step kernel runs; the step kernel (Params::gate) then returns untouched.
__global__ void check_actions_kernel(long long B, const long long *a, long long n_actions, unsigned *err) {
    bool bad = false;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += (long long)gridDim.x * blockDim.x) {
        const long long v = a[i];
        bad |= v < 0 || v >= n_actions;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, (unsigned)FLAG_BAD_ACTION);
}

// harness.first_episode_rewards (harness.py:48-61), one step's worth: an env
// that finishes its first episode records info["episode_reward"]; the
// warp-aggregated count lets the host poll one word instead of the masks.
__global__ void first_episode_kernel(long long B, const uint8_t *done, const double *ep_rew, uint8_t *seen,
                                     double *out, unsigned long long *n_seen) {
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool first = false;
    if (b < B) {
        first = done[b] && !seen[b];
        if (first) {
            out[b] = ep_rew[b];
            seen[b] = 1;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, first);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(n_seen, (unsigned long long)__popc(m));
}

// state_dict export (env.py:535-559), team per env
template <class G, int DOM>
__global__ void __launch_bounds__(256) export_kernel(const Params p, lg_state dst) {
    using Row = typename G::Row;
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    Team<G> t;
    const long long env = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G::TEAM;
    if (env >= p.B) return;
    EnvRegs<G, DOM> e;
    load_env<G, DOM>(p, t, env, e);
    const int H = p.H, W = p.W, HW = H * W;
    Bd<G> act = rect_board(t, e.h, e.w);
    Bd<G> ed = andnot(act, e.frz);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int r = t.row(k);
        if (r >= H) continue;
        cnt += popc(ed.r[k]);
        for (int c = 0; c < W; c++) {
            Row bit = Row(1) << c;
            bool a = (act.r[k] & bit) != 0;
            int tile = a ? 0 : N;
#pragma unroll
            for (int q = 0; q < NPL; q++)
                if (e.pl[q].r[k] & bit) tile = q + 1;
            size_t o = ((size_t)env * H + r) * W + c;
            dst.tiles[o] = (uint8_t)tile;
            dst.active[o] = a;
            dst.frozen[o] = (e.frz.r[k] & bit) != 0;
        }
    }
    int inc = t.scan(cnt);
    int off = inc - cnt;
    int32_t *ord = dst.order + (size_t)env * HW;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int r = t.row(k);
        if (r >= H) continue;
        Row x = ed.r[k];
        if (r & 1) {
            while (x) {
                int c = msb(x);
                x &= ~(Row(1) << c);
                ord[off++] = r * W + c;
            }
        } else {
            while (x) {
                int c = ctz(x);
                x &= x - 1;
                ord[off++] = r * W + c;
            }
        }
    }
    int total = t.from(inc, G::TEAM - 1);
    for (int i = total + t.lane; i < HW; i += G::TEAM) ord[i] = -1;
    if (t.lane != 0) return;
    dst.shape_hw[2 * env] = e.h;
    dst.shape_hw[2 * env + 1] = e.w;
    dst.order_len[env] = e.order_len;
    dst.pos_idx[env] = e.pos_idx;
    dst.pos[2 * env] = e.pr;
    dst.pos[2 * env + 1] = e.pc;
    dst.t[env] = e.t;
    dst.changes[env] = e.changes;
    dst.max_steps[env] = e.max_steps;
    for (int m = 0; m < M; m++) {
        dst.lo[(size_t)m * p.B + env] = e.lo[m];
        dst.hi[(size_t)m * p.B + env] = e.hi[m];
        dst.values[(size_t)m * p.B + env] = e.val[m];
        dst.unreach[(size_t)m * p.B + env] = (e.unr >> m) & 1;
    }
    dst.prev_loss[env] = e.prev_loss;
    dst.ep_reward[env] = e.ep_reward;
    dst.ep_start_loss[env] = e.ep_start_loss;
    dst.metric_seeds[env] = p.det ? e.mseed : p.mseed[env];
    uint64_t *rg = dst.rng + 6 * env;
    rg[0] = (uint64_t)(e.g.s >> 64);
    rg[1] = (uint64_t)e.g.s;
    rg[2] = (uint64_t)(e.g.inc >> 64);
    rg[3] = (uint64_t)e.g.inc;
    rg[4] = e.g.has;
    rg[5] = e.g.u;
}

// load_state_dict (env.py:561-585), team per env. `pos` must hold the
// current cell (the Python mirror derives it from order[pos_idx] for narrow).
template <class G, int DOM>
__global__ void __launch_bounds__(256) import_kernel(const Params p, lg_state src) {
    using Row = typename G::Row;
    constexpr int NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    Team<G> t;
    const long long env = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G::TEAM;
    if (env >= p.B) return;
    const int H = p.H, W = p.W;
    typename G::Row *rw = rows_of<G, DOM>(p, env);
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int r = t.row(k);
        Row pl[NPL > 0 ? NPL : 1], fr = 0;
        for (int q = 0; q < NPL; q++) pl[q] = 0;
        if (r < H) {
            for (int c = 0; c < W; c++) {
                size_t o = ((size_t)env * H + r) * W + c;
                int tile = src.tiles[o];
                bool a = src.active[o] != 0;
                if (a && tile >= 1 && tile <= NPL) pl[tile - 1] |= Row(1) << c;
                if (src.frozen[o]) fr |= Row(1) << c;
            }
        }
        for (int q = 0; q < NPL; q++) rw[q * G::ROWS + r] = pl[q];
        rw[NPL * G::ROWS + r] = fr;
    }
    if (t.lane != 0) return;
    Hot hv;
    uint32_t h = (uint32_t)src.shape_hw[2 * env], w = (uint32_t)src.shape_hw[2 * env + 1];
    uint32_t pr = (uint32_t)src.pos[2 * env], pc = (uint32_t)src.pos[2 * env + 1];
    hv.geo = h | (w << 8) | (pr << 16) | (pc << 24);
    hv.pos_idx = (int32_t)src.pos_idx[env];
    hv.order_len = (int32_t)src.order_len[env];
    hv.changes = (int32_t)src.changes[env];
    hv.t = src.t[env];
    hv.max_steps = src.max_steps[env];
    p.hot[env] = hv;
    int *mv = p.mv + env * 24;
    int unr = 0;
    for (int m = 0; m < 8; m++) {
        bool in = m < M;
        mv[m] = in ? (int)src.values[(size_t)m * p.B + env] : 0;
        mv[8 + m] = in ? (int)src.lo[(size_t)m * p.B + env] : 0;
        mv[16 + m] = in ? (int)src.hi[(size_t)m * p.B + env] : 0;
        if (in && src.unreach[(size_t)m * p.B + env]) unr |= 1 << m;
    }
    mv[7] = unr;
    double *lv = p.lossv + env * 4;
    lv[0] = src.prev_loss[env];
    lv[1] = src.ep_reward[env];
    lv[2] = src.ep_start_loss[env];
    lv[3] = 0.0;
    p.mseed[env] = src.metric_seeds[env];
    const uint64_t *rg = src.rng + 6 * env;
    p.rs[2 * env] = make_ulonglong2(rg[0], rg[1]);
    p.rs[2 * env + 1] = make_ulonglong2((rg[4] & 0xFFFFFFFFull) | (rg[5] << 32), 0ull);
    p.ri[env] = make_ulonglong2(rg[2], rg[3]);
}

// compute_metrics_batch on raw stacks (problems.py:105-129), team per grid.
template <class G, int DOM>
__global__ void __launch_bounds__(256) metrics_kernel(long long n, int H, int W, const uint8_t *tiles,
                                                      const uint8_t *active, uint64_t *rng,
                                                      int64_t *values, uint8_t *unreach) {
    extern __shared__ __align__(16) unsigned char smem[];
    using Row = typename G::Row;
    constexpr int NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    Team<G> t;
    const int ti = threadIdx.x / G::TEAM;
    const long long b = (long long)blockIdx.x * (blockDim.x / G::TEAM) + ti;
    if (b >= n) return;
    uint16_t *uf = reinterpret_cast<uint16_t *>(smem + (size_t)ti * G::ROWS * G::RUNS * 2);
    Bd<G> pl[NPL], act;
#pragma unroll
    for (int k = 0; k < G::RPL; k++) {
        int r = t.row(k);
        Row a = 0;
        Row q[NPL];
        for (int j = 0; j < NPL; j++) q[j] = 0;
        if (r < H) {
            for (int c = 0; c < W; c++) {
                size_t o = ((size_t)b * H + r) * W + c;
                if (active[o]) {
                    a |= Row(1) << c;
                    int tile = tiles[o];
                    if (tile >= 1 && tile <= NPL) q[tile - 1] |= Row(1) << c;
                }
            }
        }
        act.r[k] = a;
        for (int j = 0; j < NPL; j++) pl[j].r[k] = q[j];
    }
    Pcg g;
    g.s = g.inc = 0;
    g.has = g.u = 0;
    if (rng) {
        const uint64_t *rg = rng + 6 * b;
        g.s = ((u128)rg[0] << 64) | rg[1];
        g.inc = ((u128)rg[2] << 64) | rg[3];
        g.has = (uint32_t)rg[4];
        g.u = (uint32_t)rg[5];
    }
    int val[8] = {0, 0, 0, 0, 0, 0, 0, 0}, unr = 0;
    TeamK<G> k{t, low_mask<Row>(W)};
    compute_metrics<TeamK<G>, DOM>(k, pl, act, g, uf, val, unr);
    if (t.lane != 0) return;
    for (int m = 0; m < M; m++) {
        values[(size_t)m * n + b] = val[m];
        unreach[(size_t)m * n + b] = (unr >> m) & 1;
    }
    if (rng) {
        uint64_t *rg = rng + 6 * b;
        rg[0] = (uint64_t)(g.s >> 64);
        rg[1] = (uint64_t)g.s;
        rg[4] = g.has;
        rg[5] = g.u;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct lg_env {
    lg_config cfg;
    int device;
    long long B, offset;
    unsigned long long seed;
    int geo;  // 1 = solo (thread per env), 16 / 32 / 64 = lane-team row capacity
    int team, threads, E;
    int N, M, NPL, C, OH, OW;
    long long n_actions;
    size_t row_bytes, rows_per_env;
    Params base;
    size_t smem;
    // solo slot layout without the frozen plane (Params::elide): allowed by the
    // config (no pinpoints, no control planes, float32 obs, slot layout) and
    // used while every env's frozen plane equals its border plane (`plain`;
    // re-checked on device by every lg_import_state).
    bool elide_ok = false, plain = true;
    bool frz_ok = false;  // solo layout without pinpoints: Params::frz_derived while `plain`
    int slot_elide = 0;
    size_t smem_elide = 0;
    // e2e staging (lazy)
    long long *d_act = nullptr;
    void *d_obs = nullptr;
    double *d_rew = nullptr;
    unsigned char *d_done = nullptr, *d_term = nullptr;
    double *d_er = nullptr, *d_es = nullptr, *d_fl = nullptr;
    long long *d_el = nullptr;
    // the per-env outputs above are one device block [rew|er|es|fl|el|done|term]
    // (d_small); small batches copy it to the host in one transfer (h_small)
    void *d_small = nullptr;
    uint8_t *h_small = nullptr;
    // packed observation transfer (lg_step_host): device bit stream, pinned
    // host copy, one event per copied chunk
    uint32_t *d_bits = nullptr;
    uint8_t *h_bits = nullptr;
    size_t bits_bytes = 0, chunk_bytes = 0;
    std::vector<cudaEvent_t> chunk_ev;
    // chained lg_step_random launches: per-block tickets, and whether
    // the last library call on this env was a chained step on chain_stream
    unsigned *tickets = nullptr;
    long long tickets_grid = 0;
    long long *act_scratch = nullptr;  // geo 64: lg_step_random's actions when not recorded
    bool chain_live = false, pdl = false;
    cudaStream_t chain_stream = nullptr;
};

// Launch a step kernel; `pdl`: as a programmatic dependent launch of the
// previous chained step on the stream (env_kernels.cuh chain_enter).
static cudaError_t launch_step(void (*kern)(const Params, int), unsigned grid, unsigned threads, size_t smem,
                               cudaStream_t s, const Params &q, int mode, bool pdl) {
    if (!pdl) {
        kern<<<grid, threads, smem, s>>>(q, mode);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(grid);
    c.blockDim = dim3(threads);
    c.dynamicSmemBytes = smem;
    c.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    c.numAttrs = 1;
    return cudaLaunchKernelEx(&c, kern, q, mode);
}

static void fastdiv_init(FastDiv &f, uint32_t d) {
    f.d = d;
    if (d <= 1) {
        f.mul = 0;
        f.shr = 0;
        return;
    }
    uint32_t l = 0;
    while ((1ull << l) < d) l++;  // ceil(log2 d)
    uint32_t pw = 31 + l;
    f.mul = (uint32_t)(((1ull << pw) + d - 1) / d);
    f.shr = pw - 32;
}

static int dom_n(int d) { return d == 0 ? 2 : d == 1 ? 4 : 6; }
static int dom_m(int d) { return d == 0 ? 2 : d == 1 ? 4 : 7; }

template <class G, int DOM, int S>
static int launch_env_k(lg_env *e, const Params &q, int mode, cudaStream_t s) {
    CU(smem_attr((const void *)env_kernel<G, DOM, S>));
    const int E = e->threads / G::TEAM;
    const long long grid = (e->B + E - 1) / E;
    if (q.chain && grid > e->tickets_grid) {
        set_err("chained launch grid exceeds the ticket array");
        return LG_EINVAL;
    }
    CU(launch_step(env_kernel<G, DOM, S>, (unsigned)grid, e->threads, e->smem, s, q, mode, e->pdl));
    return LG_OK;
}

// Specialised lane-team kernels (env_kernels.cuh, S = spec_of(rep, no pins))
// for the BASELINE configs' (G, domain, representation) triples.
template <class G, int DOM, int S>
static constexpr bool spec_enabled() {
    return (std::is_same<G, G64>::value && DOM == 0 && S == spec_of(LG_NARROW, true)) ||  // c4
           (std::is_same<G, G16>::value && DOM == 1 && S == spec_of(LG_TURTLE, true));    // c2
}

// plain = the flags a specialised kernel fixes (no controls, no det metrics, float32 obs)
static bool plain_launch(const Params &q) {
    const char *ns = getenv("LG_NO_SPEC");
    return q.n_ctrl == 0 && !q.det && !q.obs_u8 && !q.obs_bits && !(ns && ns[0] == '1');
}

template <class G, int DOM>
static int launch_env_t(lg_env *e, const Params &p, int mode, cudaStream_t s) {
    Params q = p;
    const char *ea = getenv("LG_EARLY");
    q.early = ea ? ea[0] == '1' : 1;
    if (plain_launch(q)) {
        const bool np = q.n_pins == 0;
#define LG_TRY_SPEC(REP, NP)                                                                     \
    if constexpr (spec_enabled<G, DOM, spec_of(REP, NP)>())                                     \
        if (q.rep == REP && np == NP) return launch_env_k<G, DOM, spec_of(REP, NP)>(e, q, mode, s);
        LG_TRY_SPEC(LG_NARROW, true)
        LG_TRY_SPEC(LG_NARROW, false)
        LG_TRY_SPEC(LG_TURTLE, true)
        LG_TRY_SPEC(LG_TURTLE, false)
        LG_TRY_SPEC(LG_WIDE, true)
        LG_TRY_SPEC(LG_WIDE, false)
#undef LG_TRY_SPEC
    }
    return launch_env_k<G, DOM, 0>(e, q, mode, s);
}

template <int DOM>
static int launch_solo_t(lg_env *e, const Params &p, int mode, cudaStream_t s) {
    CU(smem_attr((const void *)SoloKernel<DOM>::fn));
    CU(smem_attr((const void *)SoloKernel<DOM>::fn_small));
    long long grid = (e->B + e->E - 1) / e->E;
    Params q = p;
    size_t smem = e->smem;
    q.frz_derived = e->frz_ok && e->plain;
    // early observation stores (solo_kernel.cuh): c5 +2.5%, its 131k-env shard
    // +14%; dungeon's larger step spills under it (c3 graph replay -1.5%)
    const char *ea = getenv("LG_EARLY");
    q.early = ea ? ea[0] == '1' : !getenv("LG_NO_EARLY");  // dungeon: compiled out (LG_DUNGEON_EARLY)
    const char *co = getenv("LG_COOP");
    q.coop = co ? co[0] == '1' : 1;
    if (e->elide_ok && e->plain && p.obs) {
        q.elide = 1;
        q.env_smem = e->slot_elide;
        smem = e->smem_elide;
    }
    constexpr int S = SoloKernel<DOM>::spec;
    const bool spec = S != 0 && plain_launch(q) && q.rep == (S & 3) - 1 && (!(S & SPEC_NOPINS) || q.n_pins == 0);
    void (*kern)(const Params, int) = e->E == e->threads ? (spec ? SoloKernel<DOM>::fn_spec : SoloKernel<DOM>::fn)
                                                         : (spec ? SoloKernel<DOM>::fn_small_spec
                                                                 : SoloKernel<DOM>::fn_small);
    if (spec) CU(smem_attr((const void *)kern));
    if (q.chain && grid > e->tickets_grid) {
        set_err("chained launch grid exceeds the ticket array");
        return LG_EINVAL;
    }
    CU(launch_step(kern, (unsigned)grid, e->threads, smem, s, q, mode, e->pdl));
    CU(cudaGetLastError());
    return LG_OK;
}

static int launch_env(lg_env *e, const Params &p, int mode, cudaStream_t s) {
    int d = e->cfg.domain;
    switch (e->geo) {
    case 1:
        return d == 0 ? launch_solo_t<0>(e, p, mode, s) : d == 1 ? launch_solo_t<1>(e, p, mode, s)
                                                                 : launch_solo_t<2>(e, p, mode, s);
    case 16:
        return d == 0 ? launch_env_t<G16, 0>(e, p, mode, s)
               : d == 1 ? launch_env_t<G16, 1>(e, p, mode, s)
                        : launch_env_t<G16, 2>(e, p, mode, s);
    case 32:
        return d == 0 ? launch_env_t<G32, 0>(e, p, mode, s)
               : d == 1 ? launch_env_t<G32, 1>(e, p, mode, s)
                        : launch_env_t<G32, 2>(e, p, mode, s);
    default:
        return d == 0 ? launch_env_t<G64, 0>(e, p, mode, s)
               : d == 1 ? launch_env_t<G64, 1>(e, p, mode, s)
                        : launch_env_t<G64, 2>(e, p, mode, s);
    }
}

template <class G, int DOM>
static int launch_state_t(lg_env *e, const Params &p, const lg_state &st, bool exp, cudaStream_t s) {
    long long threads = e->B * G::TEAM;
    unsigned grid = (unsigned)((threads + 255) / 256);
    if (exp) export_kernel<G, DOM><<<grid, 256, 0, s>>>(p, st);
    else import_kernel<G, DOM><<<grid, 256, 0, s>>>(p, st);
    CU(cudaGetLastError());
    return LG_OK;
}

template <int DOM>
static int launch_solo_state_t(lg_env *e, const Params &p, const lg_state &st, bool exp, cudaStream_t s) {
    unsigned grid = (unsigned)((e->B + 127) / 128);
    if (exp) solo_export_kernel<DOM><<<grid, 128, 0, s>>>(p, st);
    else solo_import_kernel<DOM><<<grid, 128, 0, s>>>(p, st);
    CU(cudaGetLastError());
    return LG_OK;
}

static int launch_state(lg_env *e, const lg_state &st, bool exp, cudaStream_t s) {
    int d = e->cfg.domain;
    const Params &p = e->base;
    switch (e->geo) {
    case 1:
        return d == 0 ? launch_solo_state_t<0>(e, p, st, exp, s)
               : d == 1 ? launch_solo_state_t<1>(e, p, st, exp, s)
                        : launch_solo_state_t<2>(e, p, st, exp, s);
    case 16:
        return d == 0 ? launch_state_t<G16, 0>(e, p, st, exp, s)
               : d == 1 ? launch_state_t<G16, 1>(e, p, st, exp, s)
                        : launch_state_t<G16, 2>(e, p, st, exp, s);
    case 32:
        return d == 0 ? launch_state_t<G32, 0>(e, p, st, exp, s)
               : d == 1 ? launch_state_t<G32, 1>(e, p, st, exp, s)
                        : launch_state_t<G32, 2>(e, p, st, exp, s);
    default:
        return d == 0 ? launch_state_t<G64, 0>(e, p, st, exp, s)
               : d == 1 ? launch_state_t<G64, 1>(e, p, st, exp, s)
                        : launch_state_t<G64, 2>(e, p, st, exp, s);
    }
}

static bool force_team() {
    const char *v = getenv("LG_FORCE_TEAM");
    return v && v[0] == '1';
}

static int pick_geo(int H, int W) {
    if (W <= 16 && H <= 16 && !force_team()) return 1;
    if (W <= 32 && H <= 16) return 16;
    if (W <= 32 && H <= 32) return 32;
    return 64;
}

static int validate_cfg(const lg_config *c) {
    if (!c) {
        set_err("null config");
        return LG_EINVAL;
    }
    if (c->domain < 0 || c->domain > 2) {
        set_err("unknown domain id %d", c->domain);
        return LG_EINVAL;
    }
    if (c->representation < 0 || c->representation > 2) {
        set_err("unknown representation id %d", c->representation);
        return LG_EINVAL;
    }
    if (c->max_h < 3 || c->max_w < 3 || c->max_h > 64 || c->max_w > 64) {
        set_err("max shape must be within 3..64 per side on device");
        return LG_EINVAL;
    }
    if (c->representation != LG_WIDE && (c->obs_size < 3 || c->obs_size > 128)) {
        set_err("obs_size must be within 3..128 on device");
        return LG_EINVAL;
    }
    if (c->obs_format < 0 || c->obs_format > 2) {
        set_err("unknown observation format %d", c->obs_format);
        return LG_EINVAL;
    }
    if (c->n_pins < 0 || c->n_pins > 16 || c->n_ctrl < 0 || c->n_ctrl > 7) {
        set_err("too many pinpoints or controls");
        return LG_EINVAL;
    }
    return LG_OK;
}

extern "C" int lg_create(const lg_config *cfg, int64_t n_envs, int64_t global_offset, uint64_t seed,
                         int device, lg_env **out) {
    if (validate_cfg(cfg)) return LG_EINVAL;
    if (n_envs < 1) {
        set_err("need at least one environment");
        return LG_EINVAL;
    }
    if (n_envs > (1LL << 31) - 1) {
        set_err("at most 2^31-1 environments per device");
        return LG_EINVAL;
    }
    DEVICE_GUARD(device);
    lg_env *e = new (std::nothrow) lg_env();
    if (!e) {
        set_err("out of host memory");
        return LG_ECUDA;
    }
    e->cfg = *cfg;
    e->device = device;
    e->B = n_envs;
    e->offset = global_offset;
    e->seed = seed;
    const int H = cfg->max_h, W = cfg->max_w;
    e->N = dom_n(cfg->domain);
    e->M = dom_m(cfg->domain);
    e->NPL = e->N - 1;
    e->C = e->N + 2 + cfg->n_ctrl;
    if (cfg->representation == LG_WIDE) {
        e->OH = H;
        e->OW = W;
    } else {
        e->OH = e->OW = cfg->obs_size;
    }
    e->n_actions = cfg->representation == LG_TURTLE ? 4 + e->N
                   : cfg->representation == LG_WIDE ? (long long)H * W * e->N
                                                    : e->N + 1;

    Params &p = e->base;
    memset(&p, 0, sizeof p);
    p.B = (int)n_envs;
    p.H = H;
    p.W = W;
    p.rep = cfg->representation;
    p.OH = e->OH;
    p.OW = e->OW;
    p.half = (cfg->obs_size - 1) / 2;
    p.randomize = cfg->randomize_shape;
    p.weighted = cfg->init_weighted;
    p.n_pins = cfg->n_pins;
    p.n_ctrl = cfg->n_ctrl;
    p.det = cfg->det_metrics;
    p.max_steps = cfg->max_steps;
    p.budget = cfg->change_budget;
    p.n_actions = e->n_actions;
    p.goffset = global_offset;
    for (int i = 0; i < 16; i++) p.pins[i] = cfg->pins[i];
    for (int i = 0; i < 8; i++) {
        p.ctrl[i] = cfg->ctrl[i];
        p.cdf[i] = cfg->init_cdf[i];
        p.w[i] = cfg->weights[i];
    }
    p.obs_u8 = cfg->obs_format == 1;
    p.obs_bits = cfg->obs_format == 2;
    if ((p.obs_u8 || p.obs_bits) && cfg->n_ctrl > 0) {
        set_err("uint8/bits observations need a config without controllable metrics");
        delete e;
        return LG_EINVAL;
    }
    p.OO = (uint32_t)(e->OH * e->OW);
    p.PB = (uint32_t)(e->N + 2) * p.OO;
    p.PE = (uint32_t)e->C * p.OO;
    fastdiv_init(p.divPE, p.PE);
    fastdiv_init(p.divOO, p.OO);
    p.img_words = (int)((p.PB + 31) / 32 + 1);  // + pad word for the 2-word funnel shift

    e->geo = pick_geo(H, W);
    // Batches below 19k envs on a 16x16-or-smaller map are at most one wave of
    // latency-bound work: splitting each env over a 16-lane team shortens the
    // per-env dependency chain (measured c2, 4,096 envs: 92 M vs 56 M
    // env-steps/s; c1, 64 envs: 4.7 M vs 3.5 M; 16..1,000 envs +20..35%).
    // LG_SOLO_SMALL=1 keeps them on the solo kernel (block mode).
    const char *ss = getenv("LG_SOLO_SMALL");
    const char *sm_ = getenv("LG_SOLO_MID");  // the round-1 name
    const bool solo_small = (ss && ss[0] == '1') || (sm_ && sm_[0] == '1');
    if (e->geo == 1 && n_envs < 148LL * 4 * 32 && !solo_small)
        e->geo = 16;  // lane team of 16, one row per lane (H <= 16)
    if (e->geo == 1) {
        // one env per thread; per-env shared slot (in 32-bit words): bit image +
        // 8 control floats, >= 33 words (union-find scratch), odd stride so the
        // 32 lanes of a warp hit 32 different banks.
        int slot = p.img_words + (p.n_ctrl > 0 ? 8 : 0);
        if (slot < 33) slot = 33;
        if (!(slot & 1)) slot++;
        p.env_smem = slot;
        e->team = 1;
        const char *tb = getenv("LG_SOLO_THREADS");
        // dungeon: 4-warp blocks (c3 steady state with the chained launches
        // 593 -> 608 M env-steps/s over 3 runs each); binary: 2 (equal either way)
        int warp_threads = tb ? atoi(tb) : (cfg->domain == 2 ? 128 : 64);
        if (warp_threads != 32 && warp_threads != 64 && warp_threads != 128) warp_threads = 64;
        if (n_envs >= 148LL * 4 * 32) {  // >= 4 warps per SM: each warp writes its own 32 envs
            e->threads = warp_threads;
            e->E = warp_threads;
        } else {  // small batch: E envs per block, the whole block writes
            long long per = n_envs / (148 * 4);
            int E = n_envs <= 148LL * 8 ? 4 : 8;
            while (E < 32 && E * 2 <= per) E *= 2;
            e->E = E;
            e->threads = 128;
        }
        p.solo_E = e->E;
        e->smem = (size_t)e->E * slot * 4;
        // stream layout (no control planes): one bit stream per warp. Measured
        // faster when env boundaries are word aligned (c3: +21%), slower
        // otherwise (c5: -5%, c2 block mode: -30%); LG_STREAM=0/1 overrides.
        const char *sm = getenv("LG_STREAM");
        bool want_stream = (p.PE % 32 == 0) && e->E == e->threads;
        if (sm) want_stream = sm[0] == '1';
        if (p.PB == p.PE && want_stream) {
            int G = e->E == e->threads ? 32 : e->E;
            int sw = (int)(((long long)G * p.PE + 31) / 32 + 1);
            sw = sw + sw / 32 + 1;  // swizzle pad words (sidx)
            sw = (sw + 3) & ~3;
            int gw;
            if ((int)(p.PE / 32) - 2 >= 36) {  // union-find scratch fits in each env's own words
                gw = sw;
                sw = 0;
            } else {
                gw = sw + G * 33;
            }
            gw = (gw + 3) & ~3;
            size_t bytes = (size_t)gw * 4 * (e->E == e->threads ? e->threads / 32 : 1);
            if (bytes <= 200 * 1024) {
                p.stream_mode = 1;
                p.stream_words = sw;  // 0: scratch inside the env's own stream words
                p.group_words = gw;
                e->smem = bytes;
            }
        }
        if (e->OW > 64 || e->smem > 200 * 1024) e->geo = pick_geo(17, W);  // too wide: lane teams
        e->frz_ok = e->geo == 1 && p.n_pins == 0 && !getenv("LG_NO_FRZ_DERIVE");
        if (e->geo == 1 && !p.stream_mode && p.n_ctrl == 0 && p.n_pins == 0 && !p.obs_u8 &&
            !getenv("LG_NO_ELIDE")) {
            int se = (int)((p.PB - p.OO + 31) / 32 + 1);
            if (se < 33) se = 33;
            if (!(se & 1)) se++;
            e->elide_ok = true;
            e->slot_elide = se;
            e->smem_elide = (size_t)e->E * se * 4;
        }
    }
    if (e->geo != 1) {
        e->team = e->geo == 16 ? 16 : 32;
        const char *tt = getenv("LG_TEAM_THREADS");
        // one-warp blocks, so a block's slot frees as soon as its envs are done
        // (recompute times vary): 64x64 maps, one env per block (c4 92 M vs
        // 87 M env-steps/s); 16-lane teams, two envs per block (c1 +5%, c2 +3%
        // with the chained launches); 32-row teams keep two warps
        e->threads = tt ? atoi(tt) : (e->geo == 32 ? 64 : 32);
        if (e->threads != 32 && e->threads != 64 && e->threads != 128 && e->threads != 256) e->threads = 64;
        e->E = e->threads / e->team;
        int rows = e->geo == 16 ? 16 : e->geo == 32 ? 32 : 64;
        int runs = e->geo == 64 ? 32 : 16;
        // bit image, then union-find scratch (separate: the specialised kernels
        // store part of the observation after the recompute), then control floats
        const size_t uf_bytes = ((size_t)rows * runs * 2 + 15) & ~(size_t)15;
        const size_t img_bytes = ((size_t)p.img_words * 4 + 15) & ~(size_t)15;
        const size_t scratch = img_bytes + uf_bytes;
        p.off_uf = (int)img_bytes;
        p.off_ctrl = (int)scratch;
        p.env_smem = (int)(scratch + 32);
        e->smem = (size_t)e->E * p.env_smem;
        e->row_bytes = e->geo == 64 ? 8 : 4;
        e->rows_per_env = (size_t)(e->NPL + 1) * rows;
    } else {
        e->row_bytes = 4;
        e->rows_per_env = (size_t)(e->NPL + 1) * 8;
    }
    if (e->smem > 200 * 1024) {
        set_err("observation window too large for shared memory staging");
        delete e;
        return LG_EINVAL;
    }

    size_t B = (size_t)n_envs;
    cudaError_t err = cudaSuccess;
    auto alloc = [&](void **ptr, size_t bytes) {
        if (err == cudaSuccess) err = cudaMalloc(ptr, bytes);
        if (err == cudaSuccess) err = cudaMemset(*ptr, 0, bytes);
    };
    alloc(&p.rows, B * e->rows_per_env * e->row_bytes);
    alloc((void **)&p.hot, B * sizeof(Hot));
    alloc((void **)&p.mv, B * 24 * sizeof(int));
    alloc((void **)&p.lossv, B * 4 * sizeof(double));
    alloc((void **)&p.rs, B * 2 * sizeof(ulonglong2));
    alloc((void **)&p.ri, B * sizeof(ulonglong2));
    alloc((void **)&p.mseed, B * sizeof(long long));
    alloc((void **)&p.err, sizeof(unsigned));
    alloc((void **)&p.aux, sizeof(unsigned));
    e->tickets_grid = ((long long)B + e->E - 1) / e->E;  // chained lg_step_random launches
    alloc((void **)&e->tickets, (size_t)e->tickets_grid * 2 * sizeof(unsigned));
    if (e->geo == 64) alloc((void **)&e->act_scratch, B * sizeof(long long));
    if (err != cudaSuccess) {
        set_err("CUDA allocation failed: %s", cudaGetErrorString(err));
        lg_destroy(e);
        return LG_ECUDA;
    }
    seed_kernel<<<(unsigned)((B + 255) / 256), 256>>>((long long)B, seed, global_offset, p.rs, p.ri, p.rb);
    err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        set_err("seeding failed: %s", cudaGetErrorString(err));
        lg_destroy(e);
        return LG_ECUDA;
    }
    *out = e;
    return LG_OK;
}

extern "C" int lg_destroy(lg_env *e) {
    if (!e) return LG_OK;
    DeviceGuard dg(e->device);
    Params &p = e->base;
    void *ptrs[] = {p.rows, p.hot, p.mv, p.lossv, p.rs, p.ri, p.rb, p.mseed, p.err, p.aux,
                    e->d_act, e->d_obs, e->d_small,
                    e->d_bits, e->tickets, e->act_scratch};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    if (e->h_bits) cudaFreeHost(e->h_bits);
    if (e->h_small) cudaFreeHost(e->h_small);
    for (cudaEvent_t ev : e->chunk_ev) cudaEventDestroy(ev);
    delete e;
    return LG_OK;
}

extern "C" int lg_describe(const lg_env *e, lg_desc *out) {
    if (!e || !out) {
        set_err("null argument");
        return LG_EINVAL;
    }
    out->n_envs = e->B;
    out->n_actions = (int32_t)e->n_actions;
    out->n_metrics = e->M;
    out->obs_c = e->C;
    out->obs_h = e->OH;
    out->obs_w = e->OW;
    out->team = e->team;
    // bits: the batch is one stream of ceil(B*C*OH*OW/32) u32 words (no per-env size)
    out->obs_bytes_per_env = e->base.obs_bits ? 0 : (int64_t)e->C * e->OH * e->OW * (e->base.obs_u8 ? 1 : 4);
    out->state_bytes_per_env =
        (int64_t)(e->rows_per_env * e->row_bytes + sizeof(Hot) + 24 * 4 + 32 + 16 + 16 + 8 + 8);
    return LG_OK;
}

static int check_obs_ptr(const void *obs) {
    if (obs && ((uintptr_t)obs & 15)) {
        set_err("observation buffer must be 16-byte aligned");
        return LG_EINVAL;
    }
    return LG_OK;
}

// Packed transfer is used when every observation element is a 0/1 plane
// element (no control planes); LG_HOST_EXPAND=0 forces the float32 copy.
static bool packed_ok(const lg_env *e, const void *dst) {
    if (e->cfg.n_ctrl > 0) return false;
    const char *v = getenv("LG_HOST_EXPAND");
    if (v) return v[0] != '0';
    // below ~2 MB of float32 observations the copy is latency, not bandwidth:
    // into page-locked memory the plain copy wins (c1, 64 envs: 0.61 vs
    // 0.58 M env-steps/s); into pageable memory the driver stages it through
    // its own buffer (c1: 0.29 M), and the packed stream + host expansion wins
    const size_t n = (size_t)e->B * e->C * e->OH * e->OW;
    if (n * 4 >= ((size_t)2 << 20)) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, dst) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type != cudaMemoryTypeHost;
}

// Some stream words are shared by two blocks (or lane teams): they are
// merged with atomicOr into a zeroed stream. Warp-mode solo launches own
// whole words (32 envs x PE bits), so no zeroing is needed there.
static bool packed_needs_zero(const lg_env *e) {
    const uint64_t PE = e->base.PE;
    if (e->geo != 1) return PE % 32 != 0;
    return ((uint64_t)e->E * PE) % 32 != 0;
}

static int run_mode(lg_env *e, int mode, const long long *actions, void *obs, double *reward,
                    uint8_t *done, const lg_info *info, double *stats, const uint8_t *mask, void *stream,
                    unsigned flags = 0, bool obs_bits = false, const uint64_t *rand_seed = nullptr,
                    int64_t *act_out = nullptr) {
    if (!e) {
        set_err("null env");
        return LG_EINVAL;
    }
    const bool chain_was_live = e->chain_live;
    e->chain_live = false;  // any other call on the env ends a chain of lg_step_random launches
    e->pdl = false;
    if (check_obs_ptr(obs)) return LG_EINVAL;
    if (mode == MODE_STEP && ((!actions && !rand_seed) || !reward || !done)) {
        set_err("step needs actions, reward and done buffers");
        return LG_EINVAL;
    }
    DEVICE_GUARD(e->device);
    NvtxRange nv(mode_name(mode));
    Params p = e->base;
    p.actions = actions;
    p.obs = reinterpret_cast<float *>(obs);  // uint8 bytes when obs_u8
    p.reward = reward;
    p.done = done;
    if (info) {
        p.terminal = info->terminal;
        p.ep_rew = info->episode_reward;
        p.ep_len = (long long *)info->episode_length;
        p.ep_start = info->episode_start_loss;
        p.fin_loss = info->final_loss;
    }
    p.stats = stats;
    p.reset_mask = mask;
    p.no_auto_reset = (flags & LG_STEP_NO_AUTO_RESET) ? 1 : 0;
    if (obs_bits) p.obs_bits = 1;
    if (mode == MODE_STEP && (flags & LG_STEP_VALIDATE)) {
        const long long n = e->B;
        unsigned grid = (unsigned)((n + 255) / 256);
        if (grid > 148u * 8u) grid = 148u * 8u;
        check_actions_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, actions, e->n_actions, p.err);
        CU(cudaGetLastError());
        p.gate = 1;
    }
    if (p.obs_bits && obs && packed_needs_zero(e)) {
        const size_t words = ((size_t)e->B * p.PE + 31) / 32;
        CU(cudaMemsetAsync(obs, 0, words * 4, (cudaStream_t)stream));
    }
    bool chained = false;
    if (rand_seed && e->geo == 64) {
        // 64-row lane teams (kTeamChain): the actions are drawn by their own
        // kernel and the step reads them, no chaining
        long long *a = act_out ? (long long *)act_out : e->act_scratch;
        random_actions_kernel<<<(unsigned)((e->B + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
            e->B, e->offset, *rand_seed, e->n_actions, a);
        CU(cudaGetLastError());
        p.actions = a;
        rand_seed = nullptr;
    }
    if (rand_seed) {
        p.rand_act = 1;
        p.act_seed = *rand_seed;
        p.act_out = (long long *)act_out;
        // chained (programmatic dependent) launches need every launch of the
        // env to run the same grid over the same envs, and no memset between
        // two steps (packed streams with shared boundary words)
        // (measured: c5 +3%, its 131k-env shard +13%, c3 +21%, c2 +22%; the
        // 64-row lane teams, one env per 32-thread block, lost 4% and are
        // not chained -- above)
        const char *nc = getenv("LG_NO_CHAIN");
        chained = !(p.obs_bits && obs && packed_needs_zero(e)) && !(nc && nc[0] == '1');
    }
    if (chained) {
        p.chain = 1;
        p.tickets = e->tickets;
        e->pdl = chain_was_live && e->chain_stream == (cudaStream_t)stream;
    }
    const int rc = launch_env(e, p, mode, (cudaStream_t)stream);
    e->pdl = false;
    e->chain_live = chained && rc == LG_OK;
    e->chain_stream = (cudaStream_t)stream;
    return rc;
}

extern "C" int lg_reset(lg_env *e, void *obs, void *stream) {
    return run_mode(e, MODE_RESET, nullptr, obs, nullptr, nullptr, nullptr, nullptr, nullptr, stream);
}
extern "C" int lg_reset_masked(lg_env *e, const uint8_t *mask, void *obs, void *stream) {
    return run_mode(e, MODE_RESET, nullptr, obs, nullptr, nullptr, nullptr, nullptr, mask, stream);
}
extern "C" int lg_recompute(lg_env *e, const uint8_t *mask, int reprice_only, void *stream) {
    return run_mode(e, reprice_only ? MODE_REPRICE : MODE_RECOMPUTE, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, mask, stream);
}

extern "C" int lg_observe(lg_env *e, void *obs, void *stream) {
    if (!obs) {
        set_err("observe needs an output buffer");
        return LG_EINVAL;
    }
    return run_mode(e, MODE_OBSERVE, nullptr, obs, nullptr, nullptr, nullptr, nullptr, nullptr, stream);
}
extern "C" int lg_step(lg_env *e, const int64_t *actions, void *obs, double *reward, uint8_t *done,
                       const lg_info *info, double *stats, void *stream) {
    return run_mode(e, MODE_STEP, (const long long *)actions, obs, reward, done, info, stats, nullptr,
                    stream);
}

extern "C" int lg_step_random(lg_env *e, uint64_t seed, int64_t *actions_out, void *obs, double *reward,
                              uint8_t *done, const lg_info *info, double *stats, void *stream) {
    return run_mode(e, MODE_STEP, nullptr, obs, reward, done, info, stats, nullptr, stream, 0, false, &seed,
                    actions_out);
}

extern "C" int lg_step_flags(lg_env *e, const int64_t *actions, void *obs, double *reward, uint8_t *done,
                             const lg_info *info, double *stats, uint32_t flags, void *stream) {
    return run_mode(e, MODE_STEP, (const long long *)actions, obs, reward, done, info, stats, nullptr,
                    stream, flags);
}

struct ChunkPoll {
    lg_env *e;
    bool failed;
};
static bool chunk_ready(void *ctx, size_t c) {
    ChunkPoll *cp = static_cast<ChunkPoll *>(ctx);
    cudaSetDevice(cp->e->device);
    cudaError_t r = cudaEventQuery(cp->e->chunk_ev[c]);
    if (r == cudaErrorNotReady) return false;
    if (r != cudaSuccess) cp->failed = true;  // stop waiting; reported after the sync
    return true;
}

extern "C" int lg_step_host(lg_env *e, const int64_t *actions_host, void *obs_host, double *reward_host,
                            uint8_t *done_host, const lg_info *info_host, void *stream) {
    if (!e || !actions_host || !reward_host || !done_host) {
        set_err("step_host needs actions, reward and done buffers");
        return LG_EINVAL;
    }
    DEVICE_GUARD(e->device);
    NvtxRange nv("lg_step_host");
    size_t B = (size_t)e->B;
    const size_t n_elems = B * (size_t)e->C * e->OH * e->OW;
    size_t obs_bytes = n_elems * (e->base.obs_u8 ? 1 : sizeof(float));
    const bool dev_bits = e->base.obs_bits;  // the env's own format is the packed stream
    const bool packed = obs_host && (dev_bits || packed_ok(e, obs_host));
    // Staging buffers are allocated into locals and committed to the env only
    // when every allocation succeeded, so a failed call leaves no half-set
    // state behind for the next one to launch into.
    // small batches: the per-env outputs come back in one transfer (each
    // cudaMemcpyAsync costs microseconds of latency; c1 has 8 of them)
    const size_t small_bytes = B * (5 * 8 + 2);
    const bool one_copy = small_bytes <= ((size_t)1 << 20);
    if (!e->d_act) {
        void *act = nullptr, *blk = nullptr;
        uint8_t *hs = nullptr;
        cudaError_t err = cudaMalloc(&act, B * 8);
        if (err == cudaSuccess) err = cudaMalloc(&blk, small_bytes);
        if (err == cudaSuccess && one_copy) err = cudaHostAlloc((void **)&hs, small_bytes, cudaHostAllocDefault);
        if (err != cudaSuccess) {
            if (act) cudaFree(act);
            if (blk) cudaFree(blk);
            if (hs) cudaFreeHost(hs);
            set_err("CUDA allocation failed: %s", cudaGetErrorString(err));
            return LG_ECUDA;
        }
        uint8_t *b = reinterpret_cast<uint8_t *>(blk);
        e->d_act = (long long *)act;
        e->d_small = blk;
        e->h_small = hs;
        e->d_rew = (double *)(b);
        e->d_er = (double *)(b + B * 8);
        e->d_es = (double *)(b + B * 16);
        e->d_fl = (double *)(b + B * 24);
        e->d_el = (long long *)(b + B * 32);
        e->d_done = b + B * 40;
        e->d_term = b + B * 41;
    }
    if (packed && !e->d_bits) {
        const size_t bits_bytes = ((n_elems + 31) / 32) * 4;
        const char *cm = getenv("LG_EXPAND_CHUNK_MB");
        size_t chunk = (size_t)(cm ? atof(cm) * (1 << 20) : 8.0 * (1 << 20));
        chunk = chunk < 4096 ? 4096 : (chunk & ~(size_t)63);
        const size_t nchunks = dev_bits ? 0 : (bits_bytes + chunk - 1) / chunk;
        uint32_t *d_bits = nullptr;
        uint8_t *h_bits = nullptr;
        std::vector<cudaEvent_t> evs(nchunks, nullptr);
        cudaError_t err = cudaMalloc((void **)&d_bits, bits_bytes);
        if (err == cudaSuccess && !dev_bits) err = cudaHostAlloc((void **)&h_bits, bits_bytes, cudaHostAllocDefault);
        for (size_t i = 0; i < nchunks && err == cudaSuccess; i++)
            err = cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
        if (err != cudaSuccess) {
            if (d_bits) cudaFree(d_bits);
            if (h_bits) cudaFreeHost(h_bits);
            for (cudaEvent_t ev : evs)
                if (ev) cudaEventDestroy(ev);
            set_err("CUDA allocation failed: %s", cudaGetErrorString(err));
            return LG_ECUDA;
        }
        e->bits_bytes = bits_bytes;
        e->chunk_bytes = chunk;
        e->d_bits = d_bits;
        e->h_bits = h_bits;
        e->chunk_ev = std::move(evs);
    }
    if (obs_host && !packed && !e->d_obs) CU(cudaMalloc((void **)&e->d_obs, obs_bytes));
    cudaStream_t s = (cudaStream_t)stream;
    CU(cudaMemcpyAsync(e->d_act, actions_host, B * 8, cudaMemcpyHostToDevice, s));
    lg_info di = {e->d_term, e->d_er, (int64_t *)e->d_el, e->d_es, e->d_fl};
    void *dev_obs = obs_host ? (packed ? (void *)e->d_bits : e->d_obs) : nullptr;
    int rc = run_mode(e, MODE_STEP, (const long long *)e->d_act, dev_obs, e->d_rew, e->d_done,
                      info_host ? &di : nullptr, nullptr, nullptr, stream, 0, packed);
    if (rc) return rc;
    if (dev_bits) {
        if (obs_host) CU(cudaMemcpyAsync(obs_host, e->d_bits, e->bits_bytes, cudaMemcpyDeviceToHost, s));
    } else if (packed) {  // the bit stream in chunks, one event each, so expansion overlaps the copy
        for (size_t c = 0; c < e->chunk_ev.size(); c++) {
            size_t off = c * e->chunk_bytes, len = e->bits_bytes - off;
            if (len > e->chunk_bytes) len = e->chunk_bytes;
            CU(cudaMemcpyAsync(e->h_bits + off, reinterpret_cast<uint8_t *>(e->d_bits) + off, len,
                               cudaMemcpyDeviceToHost, s));
            CU(cudaEventRecord(e->chunk_ev[c], s));
        }
    } else if (obs_host) {
        CU(cudaMemcpyAsync(obs_host, e->d_obs, obs_bytes, cudaMemcpyDeviceToHost, s));
    }
    if (one_copy && e->h_small) {
        CU(cudaMemcpyAsync(e->h_small, e->d_small, small_bytes, cudaMemcpyDeviceToHost, s));
    } else {
        CU(cudaMemcpyAsync(reward_host, e->d_rew, B * 8, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(done_host, e->d_done, B, cudaMemcpyDeviceToHost, s));
    }
    if (info_host && !(one_copy && e->h_small)) {
        if (info_host->terminal) CU(cudaMemcpyAsync(info_host->terminal, e->d_term, B, cudaMemcpyDeviceToHost, s));
        if (info_host->episode_reward)
            CU(cudaMemcpyAsync(info_host->episode_reward, e->d_er, B * 8, cudaMemcpyDeviceToHost, s));
        if (info_host->episode_length)
            CU(cudaMemcpyAsync(info_host->episode_length, e->d_el, B * 8, cudaMemcpyDeviceToHost, s));
        if (info_host->episode_start_loss)
            CU(cudaMemcpyAsync(info_host->episode_start_loss, e->d_es, B * 8, cudaMemcpyDeviceToHost, s));
        if (info_host->final_loss)
            CU(cudaMemcpyAsync(info_host->final_loss, e->d_fl, B * 8, cudaMemcpyDeviceToHost, s));
    }
    auto scatter_small = [&]() {  // the one-copy block into the caller's arrays
        if (!(one_copy && e->h_small)) return;
        const uint8_t *h = e->h_small;
        memcpy(reward_host, h, B * 8);
        memcpy(done_host, h + B * 40, B);
        if (!info_host) return;
        if (info_host->episode_reward) memcpy(info_host->episode_reward, h + B * 8, B * 8);
        if (info_host->episode_start_loss) memcpy(info_host->episode_start_loss, h + B * 16, B * 8);
        if (info_host->final_loss) memcpy(info_host->final_loss, h + B * 24, B * 8);
        if (info_host->episode_length) memcpy(info_host->episode_length, h + B * 32, B * 8);
        if (info_host->terminal) memcpy(info_host->terminal, h + B * 41, B);
    };
    if (packed && !dev_bits) {
        ChunkPoll cp{e, false};
        lg_host::expand_bits(e->h_bits, obs_host, e->base.obs_u8 ? 1 : 0, n_elems, e->chunk_bytes, chunk_ready,
                             &cp);
        CU(cudaStreamSynchronize(s));
        if (cp.failed) {
            set_err("CUDA error while copying the packed observations");
            return LG_ECUDA;
        }
        scatter_small();
        return LG_OK;
    }
    CU(cudaStreamSynchronize(s));
    scatter_small();
    return LG_OK;
}

extern "C" int lg_host_threads(void) { return lg_host::expand_threads(); }

extern "C" int lg_unpack_host(const uint32_t *bits, int64_t n_elems, void *dst, int fmt) {
    if (!bits || !dst || n_elems < 0 || (fmt != 0 && fmt != 1)) {
        set_err("unpack_host needs bits, a destination, n_elems >= 0 and fmt 0 (float32) or 1 (uint8)");
        return LG_EINVAL;
    }
    if (n_elems == 0) return LG_OK;
    const size_t bytes = ((size_t)n_elems + 7) / 8;
    lg_host::expand_bits(reinterpret_cast<const uint8_t *>(bits), dst, fmt, (size_t)n_elems,
                         (bytes + 63) & ~(size_t)63, nullptr, nullptr);
    return LG_OK;
}

template <int KC, bool BF16>
static int launch_conv1(const uint32_t *bits, long long B, int C, int OH, int OW, const float *w,
                        const float *bias, int K, void *out, int relu, int nhwc, int EB, size_t smem,
                        cudaStream_t s) {
    Conv1Div dv;
    fastdiv_init(dv.oo, (uint32_t)(OH * OW));
    fastdiv_init(dv.pw, (uint32_t)(OW - 2));
    fastdiv_init(dv.np, (uint32_t)((OH - 2) * (OW - 2)));
    fastdiv_init(dv.g, (uint32_t)((C + 3) / 4));
    auto fn = conv1_bits_kernel<KC, BF16>;
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 0, per = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, smem));
    long long grid = (long long)sms * (per > 0 ? per : 1);
    if (grid * EB > B) grid = (B + EB - 1) / EB;
    fn<<<(unsigned)grid, 256, smem, s>>>(bits, B, C, OH, OW, w, bias, K, out, relu, nhwc, EB, dv);
    CU(cudaGetLastError());
    return LG_OK;
}

// conv1 tile layout for the binary observation (C = 4): row-triple tables
static int launch_conv1_tri(const uint32_t *bits, long long B, int O, const float *w, const float *bias,
                            void *out, int relu, cudaStream_t s) {
    Conv1TriDiv dv;
    fastdiv_init(dv.p, (uint32_t)(O - 2));
    const int EB = LG_TRI_EB;
    const size_t tables = (size_t)3 * 216 * 24 * 2 + (size_t)9 * 16 * 20 * sizeof(float);
    const size_t tri = ((size_t)EB * O * (O - 2) + 15) & ~(size_t)15;
    const size_t words = ((size_t)EB * 4 * O * O + 31) / 32 + 1;
    const size_t smem = tables + tri + words * 4;
    auto fn = conv1_tri_kernel;
    CU(smem_attr((const void *)fn));
    int dev = 0, sms = 0, per = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, LG_TRI_THREADS, smem));
    long long grid = (long long)sms * (per > 0 ? per : 1);
    if (grid * EB > B) grid = (B + EB - 1) / EB;
    fn<<<(unsigned)grid, LG_TRI_THREADS, smem, s>>>(bits, B, O, w, bias, out, relu, dv);
    CU(cudaGetLastError());
    return LG_OK;
}

extern "C" int lg_conv1_bits(const uint32_t *bits, int64_t n_envs, int C, int OH, int OW, const float *weight,
                             const float *bias, int K, void *out, int out_bf16, int relu, int nhwc, void *stream) {
    if (!bits || !weight || !bias || !out || n_envs < 1) {
        set_err("conv1_bits needs bits, weight, bias and output buffers and n_envs >= 1");
        return LG_EINVAL;
    }
    if (C < 1 || C > 16 || OH < 3 || OW < 3 || K < 1 || K > 64) {
        set_err("conv1_bits supports 1 <= C <= 16, 3 <= OH, OW and 1 <= K <= 64");
        return LG_EINVAL;
    }
    if (nhwc == 2 && (K != 16 || !out_bf16 || OH != OW)) {
        set_err("conv1_bits tile layout (lg_policy_trunk input) needs K = 16, bfloat16 output, square windows");
        return LG_EINVAL;
    }
    const char *cg = getenv("LG_CONV1_GENERIC");
    if (nhwc == 2 && C == 4 && OH <= 31 && !(cg && cg[0] == '1'))  // binary's planes: row triples
        return launch_conv1_tri(bits, (long long)n_envs, OH, weight, bias, out, relu, (cudaStream_t)stream);
    const int KC = (K + 3) / 4, KCt = KC <= 4 ? 4 : KC <= 8 ? 8 : 16;
    const size_t G = (size_t)((C + 3) / 4);
    const size_t table = G * 10 * 16 * (4 * KCt + 4) * sizeof(float);  // 9 tap tables + their sum
    // envs per block iteration: 4 (fewer barriers, fuller rounds), fewer when
    // four large observations (masks + bits) do not fit in shared memory
    // (tile layout: 32 envs, so a warp's stores cover whole 512-byte runs of a block)
    int EB = nhwc == 2 ? 32 : 4;
    size_t smem = 0;
    for (; EB >= 1; EB /= 2) {
        const size_t masks = ((size_t)EB * G * OH * OW + 15) & ~(size_t)15;
        const size_t words = ((size_t)EB * C * OH * OW + 31) / 32 + 1;
        smem = table + masks + words * 4;
        if (smem <= 200 * 1024) break;
    }
    if (EB < 1) {
        set_err("conv1_bits: tables + one observation exceed shared memory (%zu bytes)", smem);
        return LG_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    long long B = (long long)n_envs;
#define LG_CONV1(KCV)                                                                                   \
    return out_bf16 ? launch_conv1<KCV, true>(bits, B, C, OH, OW, weight, bias, K, out, relu, nhwc, EB, smem, s) \
                    : launch_conv1<KCV, false>(bits, B, C, OH, OW, weight, bias, K, out, relu, nhwc, EB, smem, s)
    if (KCt == 4) LG_CONV1(4);
    if (KCt == 8) LG_CONV1(8);
    LG_CONV1(16);
#undef LG_CONV1
}

static int policy_trunk(const void *c1_tiles, int64_t n_envs, int P1, const void *w2, const float *b2, const void *w3,
                        const float *b3, const float *wh, const float *bh, int n_actions, float *logits, float *value,
                        int64_t *actions, float *logp, uint64_t seed, void *stream) {
    if (!c1_tiles || !w2 || !b2 || !w3 || !b3 || !wh || !bh || !logits || !value || n_envs < 1) {
        set_err("policy_trunk needs every buffer and n_envs >= 1");
        return LG_EINVAL;
    }
    if (P1 < 3 || P1 > 126 || n_actions < 1 || n_actions > TK_MAXNA) {
        set_err("policy_trunk supports conv1 sides 3..126 and 1..%d actions", TK_MAXNA);
        return LG_EINVAL;
    }
    const void *al[] = {c1_tiles, w2, w3};
    for (const void *q : al)
        if ((uintptr_t)q & 15) {
            set_err("policy_trunk operand blocks must be 16-byte aligned");
            return LG_EINVAL;
        }
    NvtxRange nv("lg_policy_trunk");
    CU(smem_attr((const void *)trunk_kernel_t<false>, (int)TK_SMEM));
    CU(smem_attr((const void *)trunk_kernel_t<true>, (int)TK_SMEM));
    TrunkParams tp;
    tp.c1 = reinterpret_cast<const __nv_bfloat16 *>(c1_tiles);
    tp.w2 = reinterpret_cast<const __nv_bfloat16 *>(w2);
    tp.b2 = b2;
    tp.w3 = reinterpret_cast<const __nv_bfloat16 *>(w3);
    tp.b3 = b3;
    tp.wh = wh;
    tp.bh = bh;
    tp.logits = logits;
    tp.value = value;
    tp.B = n_envs;
    tp.P1 = P1;
    tp.NA = n_actions;
    tp.actions = (long long *)actions;
    tp.logp = logp;
    tp.seed = seed;
    // Whole waves of one tile per SM, then the tail: when it fills at most
    // half the SMs it runs as half-tile CTA pairs (trunk_kernel_t<true>).
    const long long tiles = (n_envs + 127) / 128;
    int dev = 0, sms = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int nch = (P1 - 2 + TK_CW - 1) / TK_CW;
    long long tail = tiles % sms;
    const char *tt = getenv("LG_TRUNK_TAIL");
    if (nch < 2 || 2 * tail > sms || (tt && tt[0] == '0')) tail = 0;
    const long long whole = tiles - tail;
    tp.tile0 = 0;
    if (whole > 0) {
        trunk_kernel_t<false><<<(unsigned)whole, TK_THREADS, TK_SMEM, (cudaStream_t)stream>>>(tp);
        CU(cudaGetLastError());
    }
    if (tail > 0) {
        tp.tile0 = whole;
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3((unsigned)(2 * tail));
        c.blockDim = dim3(TK_THREADS);
        c.dynamicSmemBytes = TK_SMEM;
        c.stream = (cudaStream_t)stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        c.attrs = at;
        c.numAttrs = 1;
        CU(cudaLaunchKernelEx(&c, trunk_kernel_t<true>, tp));
    }
    return LG_OK;
}

extern "C" int lg_policy_trunk(const void *c1_tiles, int64_t n_envs, int P1, const void *w2, const float *b2,
                               const void *w3, const float *b3, const float *wh, const float *bh, int n_actions,
                               float *logits, float *value, void *stream) {
    return policy_trunk(c1_tiles, n_envs, P1, w2, b2, w3, b3, wh, bh, n_actions, logits, value, nullptr, nullptr, 0,
                        stream);
}

extern "C" int lg_policy_trunk_sample(const void *c1_tiles, int64_t n_envs, int P1, const void *w2, const float *b2,
                                      const void *w3, const float *b3, const float *wh, const float *bh,
                                      int n_actions, float *logits, float *value, uint64_t seed, int64_t *actions,
                                      float *logp, void *stream) {
    if (!actions || !logp) {
        set_err("policy_trunk_sample needs actions and logp buffers");
        return LG_EINVAL;
    }
    return policy_trunk(c1_tiles, n_envs, P1, w2, b2, w3, b3, wh, bh, n_actions, logits, value, actions, logp, seed,
                        stream);
}

#ifdef TK_PROF
extern "C" int lg_trunk_prof(long long *host, int n_blocks) {
    CU(cudaMemcpyFromSymbol(host, g_tk_prof, (size_t)n_blocks * 16 * sizeof(long long)));
    return LG_OK;
}
#endif

extern "C" int lg_export_state(lg_env *e, const lg_state *dst, void *stream) {
    if (!e || !dst) {
        set_err("null argument");
        return LG_EINVAL;
    }
    e->chain_live = false;
    DEVICE_GUARD(e->device);
    return launch_state(e, *dst, true, (cudaStream_t)stream);
}

extern "C" int lg_import_state(lg_env *e, const lg_state *src, void *stream) {
    if (!e || !src) {
        set_err("null argument");
        return LG_EINVAL;
    }
    e->chain_live = false;
    DEVICE_GUARD(e->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!e->frz_ok && !e->elide_ok) return launch_state(e, *src, false, s);
    // the import kernel flags envs whose frozen plane is not their border plane
    CU(cudaMemsetAsync(e->base.aux, 0, 4, s));
    int rc = launch_state(e, *src, false, s);
    if (rc != LG_OK) return rc;
    unsigned flag = 1;
    CU(cudaMemcpyAsync(&flag, e->base.aux, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    e->plain = flag == 0;
    return LG_OK;
}

extern "C" int lg_errors(lg_env *e, uint32_t *flags, void *stream) {
    if (!e || !flags) {
        set_err("null argument");
        return LG_EINVAL;
    }
    e->chain_live = false;
    DEVICE_GUARD(e->device);
    cudaStream_t s = (cudaStream_t)stream;
    CU(cudaMemcpyAsync(flags, e->base.err, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    CU(cudaMemsetAsync(e->base.err, 0, 4, s));
    return LG_OK;
}

extern "C" int lg_first_episode(int64_t n, const uint8_t *done, const double *episode_reward, uint8_t *seen,
                                double *rewards, uint64_t *n_seen, void *stream) {
    if (n < 0 || (n > 0 && (!done || !episode_reward || !seen || !rewards || !n_seen))) {
        set_err("first_episode needs done, episode_reward, seen, rewards and n_seen buffers");
        return LG_EINVAL;
    }
    if (n == 0) return LG_OK;
    first_episode_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, done, episode_reward, seen, rewards, (unsigned long long *)n_seen);
    CU(cudaGetLastError());
    return LG_OK;
}

extern "C" int lg_random_actions(lg_env *e, int64_t *actions, uint64_t seed, void *stream) {
    if (!e || !actions) {
        set_err("null argument");
        return LG_EINVAL;
    }
    e->chain_live = false;
    DEVICE_GUARD(e->device);
    random_actions_kernel<<<(unsigned)((e->B + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        e->B, e->offset, seed, e->n_actions, (long long *)actions);
    CU(cudaGetLastError());
    return LG_OK;
}

template <class G, int DOM>
static int launch_metrics_t(long long n, int H, int W, const uint8_t *tiles, const uint8_t *active,
                            uint64_t *rng, int64_t *values, uint8_t *unreach, cudaStream_t s) {
    int E = 256 / G::TEAM;
    size_t smem = (size_t)E * G::ROWS * G::RUNS * 2;
    CU(smem_attr((const void *)metrics_kernel<G, DOM>));
    metrics_kernel<G, DOM><<<(unsigned)((n + E - 1) / E), 256, smem, s>>>(n, H, W, tiles, active, rng,
                                                                           values, unreach);
    CU(cudaGetLastError());
    return LG_OK;
}

extern "C" int lg_metrics(int domain, int H, int W, int64_t n, const uint8_t *tiles, const uint8_t *active,
                          uint64_t *rng, int64_t *values, uint8_t *unreach, void *stream) {
    if (domain < 0 || domain > 2 || H < 1 || W < 1 || H > 64 || W > 64 || n < 0) {
        set_err("bad metrics arguments");
        return LG_EINVAL;
    }
    if (domain == 0 && !rng) {
        set_err("binary metrics need generators");
        return LG_EINVAL;
    }
    if (n == 0) return LG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int g = pick_geo(H, W);
    if (g == 1) {
        unsigned grid = (unsigned)((n + 127) / 128);
        size_t smem = 128 * 33 * 4;
        if (domain == 0) solo_metrics_kernel<0><<<grid, 128, smem, s>>>(n, H, W, tiles, active, rng, values, unreach);
        else if (domain == 1) solo_metrics_kernel<1><<<grid, 128, smem, s>>>(n, H, W, tiles, active, rng, values, unreach);
        else solo_metrics_kernel<2><<<grid, 128, smem, s>>>(n, H, W, tiles, active, rng, values, unreach);
        CU(cudaGetLastError());
        return LG_OK;
    }
#define LGM(GG, D) launch_metrics_t<GG, D>(n, H, W, tiles, active, rng, values, unreach, s)
    if (g == 16) return domain == 0 ? LGM(G16, 0) : domain == 1 ? LGM(G16, 1) : LGM(G16, 2);
    if (g == 32) return domain == 0 ? LGM(G32, 0) : domain == 1 ? LGM(G32, 1) : LGM(G32, 2);
    return domain == 0 ? LGM(G64, 0) : domain == 1 ? LGM(G64, 1) : LGM(G64, 2);
#undef LGM
}

extern "C" int lg_seed_streams(uint64_t seed, int64_t offset, int64_t n, uint64_t *out) {
    if (!out || n < 0) {
        set_err("bad arguments");
        return LG_EINVAL;
    }
    for (int64_t i = 0; i < n; i++) {
        Pcg g;
        seedseq_pcg(seed, true, (uint64_t)(offset + i), g);
        out[6 * i + 0] = (uint64_t)(g.s >> 64);
        out[6 * i + 1] = (uint64_t)g.s;
        out[6 * i + 2] = (uint64_t)(g.inc >> 64);
        out[6 * i + 3] = (uint64_t)g.inc;
        out[6 * i + 4] = 0;
        out[6 * i + 5] = 0;
    }
    return LG_OK;
}
