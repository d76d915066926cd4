// solo_kernel.cuh -- fused env step, one environment per thread (maps <= 16x16).
//
// Warp w of a block owns 32 consecutive environments. Each lane steps its own
// environment entirely in registers (reference _Core.step, env.py:355-393, with
// in-kernel auto-reset, env.py:391-392), then streams that environment's 0/1
// observation planes (build_observation, env.py:186-233) into its slot of the
// warp's shared-memory bit image as one sequential bit stream (no atomics, no
// zero fill). After __syncwarp the whole warp expands the 32 images -- whose
// outputs are contiguous in HBM -- into float32 with coalesced 256-bit
// streaming stores (STG.E.EF.256): each lane turns 8 bits into 8 floats per
// store. There is no block-wide barrier, so warps of the same SM interleave
// their step phases with other warps' store phases.
#pragma once
#include "env_kernels.cuh"
#include "solo.cuh"

#ifndef LG_ST_CLOBBER
#define LG_ST_CLOBBER "memory"
#endif
#ifndef LG_WRITER_U
#define LG_WRITER_U 2  // 256-bit stores in flight per lane in the float32 slot writer
#endif

namespace lg {

template <int DOM>
struct SoloEnv {
    SB pl[Dom<DOM>::NPL];
    SB frz;
    int h, w, pr, pc, pos_idx, order_len, changes;
    long long t, max_steps;
    int val[8], lo[8], hi[8];
    int unr;
    double prev_loss, ep_reward, ep_start_loss;
    Pcg g;
    long long mseed;
};

// Bit-planes plane-major: plane q (q < NPL tile planes, q == NPL frozen) of
// env b is 32 bytes at rows + (q * B + b) * 32, so a warp's 32 envs read one
// contiguous KB per plane and a step that never touches the frozen plane does
// not drag its bytes along (DRAM bursts are wider than a sector).
__device__ __forceinline__ uint32_t *solo_plane(const Params &p, long long env, int q) {
    return reinterpret_cast<uint32_t *>(p.rows) + ((size_t)q * p.B + env) * 8;
}

// Per-step state traffic is split: the "hot" part (tile planes, geometry,
// counters) is read every step; the "cold" part (metric values and targets,
// losses, RNG stream) only when the step recomputes, finishes an episode or
// renders control planes. DRAM reads interleaved with the observation write
// stream cost several times their size in write bandwidth (read/write
// turnaround; tools/store_pattern.cu), so most steps read 72 bytes per env
// instead of ~330.
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_load_hot(const Params &p, long long env, SoloEnv<DOM> &e) {
    constexpr int NPL = Dom<DOM>::NPL;
#pragma unroll
    for (int q = 0; q < NPL; q++) {
        const uint4 *rw = reinterpret_cast<const uint4 *>(solo_plane(p, env, q));
        uint4 a = rw[0], b = rw[1];
        SB &d = e.pl[q];
        d.w[0] = a.x; d.w[1] = a.y; d.w[2] = a.z; d.w[3] = a.w;
        d.w[4] = b.x; d.w[5] = b.y; d.w[6] = b.z; d.w[7] = b.w;
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
    if (p.frz_derived) {  // no active frozen cell in any env: frozen = max grid minus the episode rect
        e.frz = andnot(rect_sb(p.H, p.W), rect_sb(e.h, e.w));
    } else {
        const uint4 *rw = reinterpret_cast<const uint4 *>(solo_plane(p, env, NPL));
        uint4 a = rw[0], b = rw[1];
        SB &d = e.frz;
        d.w[0] = a.x; d.w[1] = a.y; d.w[2] = a.z; d.w[3] = a.w;
        d.w[4] = b.x; d.w[5] = b.y; d.w[6] = b.z; d.w[7] = b.w;
    }
}

// vals: also the current metric values (control planes, repricing, export);
// a recompute overwrites them, so a step only needs the targets.
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_load_cold(const Params &p, long long env, SoloEnv<DOM> &e, bool vals) {
    constexpr int M = Dom<DOM>::M;
    const int4 *mv = reinterpret_cast<const int4 *>(p.mv + env * 24);
#pragma unroll
    for (int k = 0; k < 8; k++) e.val[k] = e.lo[k] = e.hi[k] = 0;
    e.unr = 0;
    if (vals) {
        int4 a = mv[0];
        e.val[0] = a.x; e.val[1] = a.y; e.val[2] = a.z; e.val[3] = a.w;
        if (M > 4) {
            int4 b = mv[1];
            e.val[4] = b.x; e.val[5] = b.y; e.val[6] = b.z; e.unr = b.w;
        } else {
            e.unr = p.mv[env * 24 + 7];
        }
    }
    {
        int4 c = mv[2], f = mv[4];
        e.lo[0] = c.x; e.lo[1] = c.y; e.lo[2] = c.z; e.lo[3] = c.w;
        e.hi[0] = f.x; e.hi[1] = f.y; e.hi[2] = f.z; e.hi[3] = f.w;
        if (M > 4) {
            int4 d = mv[3], h2 = mv[5];
            e.lo[4] = d.x; e.lo[5] = d.y; e.lo[6] = d.z; e.lo[7] = d.w;
            e.hi[4] = h2.x; e.hi[5] = h2.y; e.hi[6] = h2.z; e.hi[7] = h2.w;
        }
    }
    const double2 *lv = reinterpret_cast<const double2 *>(p.lossv + env * 4);
    double2 l0 = lv[0], l1 = lv[1];
    e.prev_loss = l0.x;
    e.ep_reward = l0.y;
    e.ep_start_loss = l1.x;
    rng_load(p, env, e.g);
    e.mseed = det_of<S>(p) ? p.mseed[env] : 0;
}

template <int DOM, int S = 0>
__device__ __forceinline__ void solo_load(const Params &p, long long env, SoloEnv<DOM> &e) {
    solo_load_hot<DOM, S>(p, env, e);
    solo_load_cold<DOM, S>(p, env, e, true);
}

template <int DOM, int S = 0>
__device__ __forceinline__ void solo_store(const Params &p, long long env, const SoloEnv<DOM> &e, bool rows_dirty,
                           bool planes_dirty, bool metrics_dirty, bool rng_dirty, bool cold = true) {
    constexpr int NPL = Dom<DOM>::NPL;
    if (rows_dirty || planes_dirty) {
#pragma unroll
        for (int q = 0; q <= NPL; q++) {
            if (q == NPL && !rows_dirty) break;
            const SB &d = q < NPL ? e.pl[q] : e.frz;
            uint4 *rw = reinterpret_cast<uint4 *>(solo_plane(p, env, q));
            rw[0] = make_uint4(d.w[0], d.w[1], d.w[2], d.w[3]);
            rw[1] = make_uint4(d.w[4], d.w[5], d.w[6], d.w[7]);
        }
    }
    Hot hv;
    hv.geo = (uint32_t)e.h | ((uint32_t)e.w << 8) | ((uint32_t)e.pr << 16) | ((uint32_t)e.pc << 24);
    hv.pos_idx = e.pos_idx;
    hv.order_len = e.order_len;
    hv.changes = e.changes;
    hv.t = e.t;
    hv.max_steps = e.max_steps;
    p.hot[env] = hv;
    constexpr int M = Dom<DOM>::M;
    // metric values + unreachable mask: one whole 32-byte sector (ints 0..7),
    // so the write needs no DRAM read-fill; the targets (lo/hi) change only
    // when an episode starts (rows_dirty) and are written only then.
    if (metrics_dirty) {
        int4 *mv = reinterpret_cast<int4 *>(p.mv + env * 24);
        mv[0] = make_int4(e.val[0], e.val[1], M > 2 ? e.val[2] : 0, M > 3 ? e.val[3] : 0);
        mv[1] = make_int4(M > 4 ? e.val[4] : 0, M > 5 ? e.val[5] : 0, M > 6 ? e.val[6] : 0, e.unr);
        if (rows_dirty) {
            mv[2] = make_int4(e.lo[0], e.lo[1], e.lo[2], e.lo[3]);
            mv[3] = make_int4(e.lo[4], e.lo[5], e.lo[6], e.lo[7]);
            mv[4] = make_int4(e.hi[0], e.hi[1], e.hi[2], e.hi[3]);
            mv[5] = make_int4(e.hi[4], e.hi[5], e.hi[6], e.hi[7]);
        }
    }
    double2 *lv = reinterpret_cast<double2 *>(p.lossv + env * 4);
    if (cold) {  // the whole 32-byte record (metrics_dirty implies cold)
        lv[0] = make_double2(e.prev_loss, e.ep_reward);
        lv[1] = make_double2(e.ep_start_loss, 0.0);
    }
    if (rng_dirty) {
        rng_store(p, env, e.g);
        if (det_of<S>(p)) p.mseed[env] = e.mseed;
    }
}

template <int DOM, int S = 0>
__device__ __forceinline__ void solo_recompute(const Params &p, SoloEnv<DOM> &e, void *uf, bool reset) {
    SoloK k;
    SB act = rect_sb(e.h, e.w);
    // _metric_rngs (env.py:327-330): the env stream, or a fresh default_rng(metric_seed)
    Pcg mg = e.g;
    if (det_of<S>(p)) seedseq_pcg((uint64_t)e.mseed, false, 0, mg);
    compute_metrics<SoloK, DOM>(k, e.pl, act, mg, uf, e.val, e.unr);
    if (!det_of<S>(p)) e.g = mg;
    double l = loss_of<DOM>(p, e.val, e.unr, e.lo, e.hi);
    e.prev_loss = l;
    if (reset) {
        e.ep_reward = 0.0;
        e.ep_start_loss = l;
    }
}

// first editable cell (row-major r*16+c) in boustrophedon order at or after row r0; -1 if none
__device__ __forceinline__ int solo_serp_first(const SB &ed, int r0) {
    int res = -1;
#pragma unroll
    for (int r = 15; r >= 0; r--) {
        uint32_t x = (r & 1) ? (ed.w[r >> 1] >> 16) : (ed.w[r >> 1] & 0xFFFFu);
        if (r >= r0 && x) res = r * 16 + ((r & 1) ? (31 - __clz((int)x)) : (__ffs((int)x) - 1));
    }
    return res;
}

__device__ __forceinline__ int solo_serp_next(const SB &ed, int r, int c) {
    uint32_t x = ed.row(r);
    if (r & 1) {
        x &= (1u << c) - 1u;
        if (x) return r * 16 + 31 - __clz((int)x);
    } else {
        x &= ~((2u << c) - 1u);
        if (x) return r * 16 + __ffs((int)x) - 1;
    }
    return solo_serp_first(ed, r + 1);
}

// set tile id `tile` (0..N-1) at (r, c) in the stored planes
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_set_tile(SoloEnv<DOM> &e, int r, int c, int tile) {
    constexpr int NPL = Dom<DOM>::NPL;
    const int wi = r >> 1;
    const uint32_t bit = 1u << ((r & 1) * 16 + c);
#pragma unroll
    for (int q = 0; q < NPL; q++)
#pragma unroll
        for (int k = 0; k < 8; k++)
        {  // value select, not a conditional store (keeps the planes in registers)
            const uint32_t m = (k == wi) ? bit : 0u;
            e.pl[q].w[k] = (e.pl[q].w[k] & ~m) | (q == tile - 1 ? m : 0u);
        }
}

// reset_rows for one env minus its final _recompute (env.py:284-325)
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_reset_setup(const Params &p, SoloEnv<DOM> &e) {
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    Pcg &g = e.g;
    int h = p.H, w = p.W;
    if (p.randomize) {  // sample_shape: width then height (grid.py:124-125)
        w = (int)pcg_integers(g, 3, p.W + 1);
        h = (int)pcg_integers(g, 3, p.H + 1);
    }
    e.h = h;
    e.w = w;
    SB act = rect_sb(h, w);
#pragma unroll
    for (int q = 0; q < NPL; q++) e.pl[q] = SB::zero();
    e.frz = andnot(rect_sb(p.H, p.W), act);
    if (p.weighted) {  // init_random: choice(n_tiles, (h, w), p), row-major (grid.py:169-191)
#pragma unroll 1
        for (int r = 0; r < 16; r++) {
            if (r < h) {
                uint32_t rowbits[NPL];
#pragma unroll
                for (int q = 0; q < NPL; q++) rowbits[q] = 0;
                for (int c = 0; c < w; c++) {
                    double u = pcg_double(g);
                    int idx = 0;
#pragma unroll
                    for (int q = 0; q < N; q++) idx += (p.cdf[q] <= u) ? 1 : 0;  // searchsorted right
                    idx = idx < N - 1 ? idx : N - 1;
#pragma unroll
                    for (int q = 0; q < NPL; q++) rowbits[q] |= (q == idx - 1) ? (1u << c) : 0u;
                }
#pragma unroll
                for (int q = 0; q < NPL; q++)
#pragma unroll
                    for (int k = 0; k < 8; k++)  // select chain keeps the register index static
                        e.pl[q].w[k] |= (k == (r >> 1)) ? (rowbits[q] << ((r & 1) * 16)) : 0u;
            }
        }
    }
    if (npins_of<S>(p) > 0) {  // place_pinpoints: Floyd over the h*w free cells (grid.py:194-225)
        int pop = h * w, k = p.n_pins;
        if (pop < k) {
            atomicOr(p.err, (unsigned)FLAG_PINPOINTS);
        } else {
            int picks[16];
            for (int j = pop - k; j < pop; j++) {
                int val = (int)pcg_bounded(g, (uint64_t)j);
                bool seen = false;
                for (int i = 0; i < j - (pop - k); i++) seen |= picks[i] == val;
                picks[j - (pop - k)] = seen ? j : val;
            }
            for (int i = k - 1; i > 0; i--) {
                int j = (int)pcg_bounded(g, (uint64_t)i);
                int tmp = picks[i];
                picks[i] = picks[j];
                picks[j] = tmp;
            }
            for (int i = 0; i < k; i++) {
                int r = picks[i] / w, c = picks[i] - (picks[i] / w) * w;
                solo_set_tile<DOM, S>(e, r, c, p.pins[i]);
                const int wi = r >> 1;
                const uint32_t bit = 1u << ((r & 1) * 16 + c);
#pragma unroll
                for (int kk = 0; kk < 8; kk++)
                    e.frz.w[kk] |= (kk == wi) ? bit : 0u;
            }
        }
    }
    int cap = h * w;  // default_targets + sample_control_targets (problems.py:48-90)
#pragma unroll
    for (int m = 0; m < M; m++) {
        int lo = 1, hi = 1;
        if (m == 0) lo = hi = cap;
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
        for (int q = 0; q < 8; q++) {
            e.lo[q] = (q == m) ? lo : e.lo[q];
            e.hi[q] = (q == m) ? hi : e.hi[q];
        }
    }
    if (det_of<S>(p)) e.mseed = (long long)pcg_bounded(g, 0x7FFFFFFFFFFFFFFFULL);  // env.py:302-303
    SB ed = andnot(act, e.frz);  // _install_row (env.py:307-325)
    e.order_len = ed.count();
    int first = solo_serp_first(ed, 0);
    if (first < 0) {
        atomicOr(p.err, (unsigned)FLAG_NO_EDITABLE);
        first = 0;
    }
    e.pr = first >> 4;
    e.pc = first & 15;
    e.pos_idx = 0;
    e.t = 0;
    e.changes = 0;
    e.max_steps = p.max_steps > 0 ? p.max_steps : 3LL * cap;
    // the caller runs _recompute(reset=True) (env.py:305)
}

// Sequential bit writer into one env's image slot.
// Stream-mode shared-memory index: one pad word after every 32 words so that
// the 32 lanes of a warp, each writing its own env's stretch of the stream,
// spread over the banks instead of colliding (env stretches are ~PE/32 words).
__device__ __forceinline__ uint32_t sidx(uint32_t w) { return w + (w >> 5); }

struct BitW {
    uint32_t *dst;
    uint32_t widx;
    uint64_t acc;
    int n;
    // stream mode: this env's bits start mid-word inside a warp-wide bit
    // stream; the first and a partial last word are shared with neighbouring
    // envs (rendered by other lanes) and are merged with atomicOr.
    bool stream, first, last;
#ifdef LG_CHECKS
    uint32_t lim = 0xFFFFFFFFu;  // words of the slot / stream (checked builds)
#endif
    __device__ __forceinline__ void emit(uint32_t word) {
#ifdef LG_CHECKS
        LG_DCHECK((stream ? sidx(widx) : widx) < lim);
#endif
        if (stream) {
            if (first) atomicOr(&dst[sidx(widx)], word);
            else dst[sidx(widx)] = word;
        } else {
            dst[widx] = word;
        }
        first = false;
        widx++;
    }
    __device__ __forceinline__ void put32(uint32_t v, int cnt) {  // cnt <= 32, v < 2^cnt
        acc |= (uint64_t)v << n;
        n += cnt;
        if (n >= 32) {
            emit((uint32_t)acc);
            acc >>= 32;
            n -= 32;
        }
    }
    __device__ __forceinline__ void put(uint64_t v, int cnt) {  // cnt <= 64
        if (cnt > 32) {
            put32((uint32_t)v, 32);
            put32((uint32_t)(v >> 32), cnt - 32);
        } else {
            put32((uint32_t)v, cnt);
        }
    }
    __device__ __forceinline__ void fill(bool one, int cnt) {
        while (cnt > 0) {
            int take = cnt < 32 ? cnt : 32;
            put32(one ? (take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1u)) : 0u, take);
            cnt -= take;
        }
    }
    __device__ __forceinline__ void flush() {
        if (stream) {
            if (n > 0) {
                if (first || !last) atomicOr(&dst[sidx(widx)], (uint32_t)acc);
                else dst[sidx(widx)] = (uint32_t)acc;
            }
            return;
        }
        if (n > 0) dst[widx++] = (uint32_t)acc;
        dst[widx++] = 0u;  // pad word read by the 2-word funnel shift
    }
};

// Render one env's 0/1 observation planes as a bit stream: into its private
// slot (slot mode), or at bit offset `bit0` of the warp/block stream whose
// bits are the concatenated outputs of consecutive envs (stream mode).
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_render(const Params &p, const SoloEnv<DOM> &e, uint32_t *slot, bool stream, uint32_t bit0,
                            bool last) {
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL;
    const int OH = p.OH, OW = p.OW, H = p.H, W = p.W;
    int r0 = 0, c0 = 0;
    if (rep_of<S>(p) != REP_WIDE) {
        r0 = e.pr - p.half;
        c0 = e.pc - p.half;
    }
    const int jlo = c0 < 0 ? -c0 : 0;
    const int jhi = (W - c0) < OW ? (W - c0) : OW;
    const uint64_t full = OW >= 64 ? ~0ull : ((1ull << OW) - 1ull);
    const uint64_t inside = (jhi > jlo ? (jhi >= 64 ? ~0ull : ((1ull << jhi) - 1ull)) : 0ull) &
                            ~((1ull << jlo) - 1ull);
    int before = -r0;
    before = before < 0 ? 0 : (before > OH ? OH : before);
    int g_lo = r0 > 0 ? r0 : 0, g_hi = (r0 + OH) < H ? (r0 + OH) : H;
    int n_in = g_hi > g_lo ? g_hi - g_lo : 0;
    int after = OH - before - n_in;
    BitW bw{slot, stream ? (bit0 >> 5) : 0u, 0, stream ? (int)(bit0 & 31) : 0, stream, true, last};
#ifdef LG_CHECKS
    bw.lim = stream ? (uint32_t)(p.stream_words > 0 ? p.stream_words : p.group_words) : (uint32_t)p.env_smem;
#endif
    const uint32_t wm = mask16(W), am = mask16(e.w);
    // plane loop kept rolled (instruction-cache footprint). The stored plane
    // for `pl` is picked with an AND/OR mask, not a select: a select chain gets
    // rewritten into a dynamically indexed load, demoting the planes to local memory.
    const int planes = N + 2 - p.elide;
#pragma unroll 1
    for (int pl = 0; pl < planes; pl++) {
        const bool fill = pl >= N;  // border and frozen planes read 1 outside the max grid
        bw.fill(fill, before * OW);
        SB cur;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t any = 0, sel = 0;
#pragma unroll
            for (int q = 0; q < NPL; q++) {
                any |= e.pl[q].w[k];
                sel |= e.pl[q].w[k] & (0u - (uint32_t)(q == pl - 1));
            }
            const uint32_t act2 = ((2 * k < e.h) ? am : 0u) | ((2 * k + 1 < e.h) ? (am << 16) : 0u);
            const uint32_t wm2 = wm | (wm << 16);
            cur.w[k] = pl == 0 ? (act2 & ~any) : pl < N ? sel : pl == N ? (~act2 & wm2) : e.frz.w[k];
        }
#pragma unroll
        for (int gr = 0; gr < 16; gr++) {
            int i = gr - r0;
            if (gr < H && i >= 0 && i < OH) {
                uint32_t m = ((gr & 1) ? (cur.w[gr >> 1] >> 16) : cur.w[gr >> 1]) & 0xFFFFu;
                uint64_t win = c0 >= 0 ? ((uint64_t)m >> c0) : ((uint64_t)m << (-c0));
                win = (win & inside) | (fill ? (full & ~inside) : 0ull);
                bw.put(win, OW);
            }
        }
        bw.fill(fill, after * OW);
    }
    bw.flush();
    if (stream) return;  // stream mode is only used without control planes
    // control planes: (value - (lo+hi)/2) / cap, float64 -> float32 (env.py:224-232)
    float *ctrl = reinterpret_cast<float *>(slot + p.img_words);
    for (int j = 0; j < nctrl_of<S>(p); j++) {
        int m = p.ctrl[j];
        int vm = 0, lm = 0, hm = 0;
#pragma unroll
        for (int q = 0; q < 8; q++)
            if (q == m) {
                vm = e.val[q];
                lm = e.lo[q];
                hm = e.hi[q];
            }
        double tgt = __ddiv_rn(__dadd_rn((double)lm, (double)hm), 2.0);
        ctrl[j] = __double2float_rn(__ddiv_rn(__dsub_rn((double)vm, tgt), (double)(e.h * e.w)));
    }
}

__device__ __forceinline__ float solo_elem(const Params &p, const uint32_t *wimg, uint32_t el, uint32_t le) {
    const uint32_t *slot = wimg + (size_t)el * p.env_smem;
    if (le < p.PB) {
        if (p.elide && le >= p.PB - p.OO) le -= p.OO;  // frozen plane == border plane
        return ((slot[le >> 5] >> (le & 31)) & 1u) ? 1.0f : 0.0f;
    }
    return reinterpret_cast<const float *>(slot + p.img_words)[fdiv(p.divOO, le - p.PB)];
}

__device__ __forceinline__ void st_cs_v8(float *ptr, const float *v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : LG_ST_CLOBBER);
}

// Expand the warp's 32 images to float32. VEC = 8 (32-byte stores) or 4.
// Each lane keeps U independent (env, element) cursors so that U stores and
// their shared-memory reads are in flight per lane (the store's source
// registers stay locked until the LSU has read them).
template <int VEC, int U>
__device__ void solo_write(const Params &p, const uint32_t *wimg, long long env0, int nenv, int lane,
                           int nthr) {
    float *out = p.obs + (size_t)env0 * p.PE;
    const uint32_t total = (uint32_t)nenv * p.PE;
    const uint32_t nv = total / VEC;
    uint32_t el[U], le[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        uint32_t e = (uint32_t)(lane + nthr * u) * VEC;
        el[u] = fdiv(p.divPE, e);
        le[u] = e - el[u] * p.PE;
    }
    const uint32_t STEP = (uint32_t)nthr * U * VEC;
    for (uint32_t q0 = lane; q0 < nv; q0 += nthr * U) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t q = q0 + nthr * u;
            if (q < nv) {
                float v[VEC];
                if (le[u] + (VEC - 1) < p.PB) {
                    const uint32_t *slot = wimg + (size_t)el[u] * p.env_smem;
                    uint32_t wi = le[u] >> 5;
                    uint32_t x = __funnelshift_r(slot[wi], slot[wi + 1], le[u] & 31);
#pragma unroll
                    for (int k = 0; k < VEC; k++) v[k] = ((x >> k) & 1u) ? 1.0f : 0.0f;
                } else {
#pragma unroll
                    for (int k = 0; k < VEC; k++) {
                        uint32_t l2 = le[u] + k, e2 = el[u];
                        if (l2 >= p.PE) {
                            l2 -= p.PE;
                            e2++;
                        }
                        v[k] = solo_elem(p, wimg, e2, l2);
                    }
                }
                if constexpr (VEC == 8) {
                    st_cs_v8(out + (size_t)q * 8, v);
                } else {
                    __stcs(reinterpret_cast<float4 *>(out) + q, make_float4(v[0], v[1], v[2], v[3]));
                }
            }
            uint32_t l = le[u] + STEP;
            uint32_t k = fdiv(p.divPE, l);
            el[u] += k;
            le[u] = l - k * p.PE;
        }
    }
    for (uint32_t t = nv * VEC + lane; t < total; t += nthr) {
        uint32_t e2 = fdiv(p.divPE, t);
        out[t] = solo_elem(p, wimg, e2, t - e2 * p.PE);
    }
}

// Branch-light writer for observations without control planes (PB == PE),
// 32-byte aligned output: U independent 256-bit stores per lane per round.
// A group of 8 elements that straddles an env boundary takes its high bits
// from the first word of the next env's image.
// [qa, qb): the range of 8-element groups to write (qa a multiple of nthr * U);
// the ragged end (groups past the last full round, elements past the last
// group) is written by the call whose range ends at the last group.
template <int U>
__device__ void solo_write_noctrl(const Params &p, const uint32_t *wimg, long long env0, int nenv, int lane,
                                  int nthr, uint32_t qa = 0, uint32_t qb = 0xFFFFFFFFu) {
    float *out = p.obs + (size_t)env0 * p.PE;
    const uint32_t PE = p.PE, stride = (uint32_t)p.env_smem;
    const uint32_t total = (uint32_t)nenv * PE;
    const uint32_t nv = total / 8;
    if (qb > nv) qb = nv;
    const uint32_t STEP = (uint32_t)nthr * U * 8;  // elements per round per lane
    uint32_t el[U], le[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        uint32_t e = (qa + (uint32_t)(lane + nthr * u)) * 8;
        el[u] = fdiv(p.divPE, e);
        le[u] = e - el[u] * PE;
    }
    const bool small_env = PE <= STEP;  // more than one wrap per round: use the divider
    // elided frozen plane: elements [PF, PE) read the border plane [PF-OO, PF)
    const uint32_t OO = p.OO, PF = p.elide ? PE - OO : PE;
    uint32_t q0 = qa + lane;
#ifdef LG_EXP_UNROLL
#pragma unroll LG_EXP_UNROLL
#endif
    for (; q0 + (uint32_t)nthr * (U - 1) < qb; q0 += (uint32_t)nthr * U) {
        uint32_t x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t *sl = wimg + el[u] * stride;
            const uint32_t b = le[u] >= PF ? le[u] - OO : le[u];
            const uint32_t wi = b >> 5;
            uint32_t v = __funnelshift_r(sl[wi], sl[wi + 1], b & 31);
            const uint32_t kf = PF - le[u];
#ifndef LG_EXP_NOSTRADDLE
            if (kf < 8) {  // group straddles the start of the (elided) frozen plane
                const uint32_t b2 = PF - OO, w2 = b2 >> 5;
                const uint32_t v2 = __funnelshift_r(sl[w2], sl[w2 + 1], b2 & 31);
                const uint32_t m = (1u << kf) - 1u;
                v = (v & m) | ((v2 << kf) & ~m);
            }
            const uint32_t k = PE - le[u];
            if (k < 8) {
                uint32_t m = (1u << k) - 1u;
                v = (v & m) | ((sl[stride] << k) & ~m);
            }
#endif
            x[u] = v;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; j++) f[j] = ((x[u] >> j) & 1u) ? 1.0f : 0.0f;
            st_cs_v8(out + (size_t)(q0 + (uint32_t)nthr * u) * 8, f);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint32_t l = le[u] + STEP;
            if (small_env) {
                uint32_t kk = fdiv(p.divPE, l);
                el[u] += kk;
                le[u] = l - kk * PE;
            } else if (l >= PE) {
                el[u] += 1;
                le[u] = l - PE;
            } else {
                le[u] = l;
            }
        }
    }
    if (qb < nv) return;
    for (uint32_t t = q0 * 8; t < total; t += (uint32_t)nthr * 8) {  // ragged end, element by element
        for (uint32_t j = 0; j < 8 && t + j < total; j++) {
            uint32_t e2 = fdiv(p.divPE, t + j);
            out[t + j] = solo_elem(p, wimg, e2, t + j - e2 * PE);
        }
    }
}

__device__ __forceinline__ void st_cs_v8u(uint8_t *ptr, const uint32_t *v) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : LG_ST_CLOBBER);
}

// uint8 observation writer (opt-in, no control planes), slot layout: 32
// elements -> 32 bytes per lane per 256-bit store, 16 with 16-byte stores.
template <int GRP>
__device__ void solo_write_u8(const Params &p, const uint32_t *wimg, long long env0, int nenv, int lane,
                              int nthr) {
    uint8_t *out = reinterpret_cast<uint8_t *>(p.obs) + (size_t)env0 * p.PE;
    const uint32_t PE = p.PE, stride = (uint32_t)p.env_smem;
    const uint32_t total = (uint32_t)nenv * PE;
    const uint32_t ng = total / GRP;
    uint32_t e0 = (uint32_t)lane * GRP;
    uint32_t el = fdiv(p.divPE, e0), le = e0 - el * PE;
    for (uint32_t q = lane; q < ng; q += nthr) {
        const uint32_t *sl = wimg + el * stride;
        uint32_t x = __funnelshift_r(sl[le >> 5], sl[(le >> 5) + 1], le & 31);
        const uint32_t k = PE - le;
        if (k < GRP) {  // group runs into the next env's image
            uint32_t m = (1u << k) - 1u;
            x = (x & m) | ((sl[stride] << k) & ~m);
        }
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < GRP / 4; i++) w[i] = bits_to_bytes4(x >> (4 * i));
        if constexpr (GRP == 32) st_cs_v8u(out + (size_t)q * 32, w);
        else __stcs(reinterpret_cast<uint4 *>(out) + q, make_uint4(w[0], w[1], w[2], w[3]));
        uint32_t l = le + (uint32_t)nthr * GRP;
        uint32_t kk = fdiv(p.divPE, l);
        el += kk;
        le = l - kk * PE;
    }
    for (uint32_t t = ng * GRP + lane; t < total; t += nthr) {
        uint32_t e2 = fdiv(p.divPE, t), l2 = t - e2 * PE;
        out[t] = (wimg[e2 * stride + (l2 >> 5)] >> (l2 & 31)) & 1u;
    }
}

// uint8 writer for the stream layout: stream word q is elements [32q, 32q+32).
__device__ void solo_write_stream_u8(const Params &p, const uint32_t *st, long long env0, int nenv, int lane,
                                     int nthr) {
    uint8_t *out = reinterpret_cast<uint8_t *>(p.obs) + (size_t)env0 * p.PE;
    const uint32_t total = (uint32_t)nenv * p.PE;
    const uint32_t ng = total / 32;
    for (uint32_t q = lane; q < ng; q += nthr) {
        uint32_t x = st[sidx(q)];
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; i++) w[i] = bits_to_bytes4(x >> (4 * i));
        st_cs_v8u(out + (size_t)q * 32, w);
    }
    for (uint32_t t = ng * 32 + lane; t < total; t += nthr) out[t] = (st[sidx(t >> 5)] >> (t & 31)) & 1u;
}

// Writer for the stream layout: the group's outputs are one bit stream, so a
// VEC-element group q is bits [q*VEC, q*VEC+VEC) -- one shared-memory word,
// a lane-constant shift, VEC selects and one store. No env bookkeeping.
template <int VEC, int U>
__device__ void solo_write_stream(const Params &p, const uint32_t *st, long long env0, int nenv, int lane,
                                  int nthr, uint32_t qa = 0, uint32_t qb = 0xFFFFFFFFu) {
    float *out = p.obs + (size_t)env0 * p.PE;
    const uint32_t total = (uint32_t)nenv * p.PE;
    const uint32_t nv = total / VEC;
    if (qb > nv) qb = nv;
    const uint32_t sh = ((uint32_t)lane * VEC) & 31;  // nthr * VEC is a multiple of 32 (and qa * VEC)
    uint32_t q0 = qa + lane;
    for (; q0 + (uint32_t)nthr * (U - 1) < qb; q0 += (uint32_t)nthr * U) {
        uint32_t x[U];
#pragma unroll
        for (int u = 0; u < U; u++) x[u] = st[sidx(((q0 + (uint32_t)nthr * u) * VEC) >> 5)] >> sh;
#pragma unroll
        for (int u = 0; u < U; u++) {
            float f[8];
#pragma unroll
            for (int j = 0; j < VEC; j++) f[j] = ((x[u] >> j) & 1u) ? 1.0f : 0.0f;
            const size_t q = q0 + (size_t)nthr * u;
            if constexpr (VEC == 8) st_cs_v8(out + q * 8, f);
            else __stcs(reinterpret_cast<float4 *>(out) + q, make_float4(f[0], f[1], f[2], f[3]));
        }
    }
    if (qb < nv) return;
    for (uint32_t q = q0; q < nv; q += nthr) {
        uint32_t x = st[sidx((q * VEC) >> 5)] >> sh;
        float f[8];
#pragma unroll
        for (int j = 0; j < VEC; j++) f[j] = ((x >> j) & 1u) ? 1.0f : 0.0f;
        if constexpr (VEC == 8) st_cs_v8(out + (size_t)q * 8, f);
        else __stcs(reinterpret_cast<float4 *>(out) + q, make_float4(f[0], f[1], f[2], f[3]));
    }
    for (uint32_t t = nv * VEC + lane; t < total; t += nthr) out[t] = ((st[sidx(t >> 5)] >> (t & 31)) & 1u) ? 1.0f : 0.0f;
}

// ---------------------------------------------------------------------------
// Packed observation transfer (lg_step_host): the 0/1 planes of the whole
// batch as ONE bit stream, element t of the float32 [B,C,OH,OW] observation
// = bit t (word t/32, bit t%32). The host library expands it to the caller's
// float32/uint8 array, so PCIe carries 1 bit per element instead of 32.
// Words that straddle a block's range boundary are shared with the
// neighbouring block and merged with atomicOr into a zeroed buffer (the host
// zeroes it when such words exist); words at the ends of the batch are private.
// ---------------------------------------------------------------------------

// local stream bits [lpos, min(lpos + 32, lend)) of the group's slot images
// (bit j of the result = local bit lpos + j), with the elided frozen plane
// read from the border plane as in solo_write_noctrl.
__device__ __forceinline__ uint32_t solo_bits32(const Params &p, const uint32_t *wimg, uint32_t lpos, uint32_t lend) {
    const uint32_t PE = p.PE, OO = p.OO, PF = p.elide ? PE - OO : PE, stride = (uint32_t)p.env_smem;
    uint32_t el = fdiv(p.divPE, lpos), le = lpos - el * PE;
    uint32_t acc = 0, got = 0;
    while (got < 32 && lpos < lend) {
        const uint32_t seg_end = le < PF ? PF : PE;
        uint32_t take = 32 - got;
        if (seg_end - le < take) take = seg_end - le;
        if (lend - lpos < take) take = lend - lpos;
        const uint32_t phys = le >= PF ? le - OO : le;
        const uint32_t *sl = wimg + el * stride;
        uint32_t bits = __funnelshift_r(sl[phys >> 5], sl[(phys >> 5) + 1], phys & 31);
        if (take < 32) bits &= (1u << take) - 1u;
        acc |= bits << got;
        got += take;
        lpos += take;
        le += take;
        if (le == PE) {
            el++;
            le = 0;
        }
    }
    return acc;
}

__device__ __forceinline__ void put_bits_word(const Params &p, uint32_t *out, unsigned long long w, uint32_t v,
                                              bool shared) {
    if (shared) atomicOr(out + w, v);
    else out[w] = v;
}

// slot layout: envs [env0, env0 + nenv) -> stream bits [env0*PE, (env0+nenv)*PE)
__device__ void solo_write_bits(const Params &p, const uint32_t *wimg, long long env0, int nenv, int lane, int nthr) {
    uint32_t *out = reinterpret_cast<uint32_t *>(p.obs);
    const unsigned long long g0 = (unsigned long long)env0 * p.PE;
    const uint32_t TB = (uint32_t)nenv * p.PE, sh = (uint32_t)(g0 & 31);
    const unsigned long long w0 = g0 >> 5;
    const uint32_t nw = (sh + TB + 31) >> 5;
    const bool at_end = env0 + nenv >= p.B;
    for (uint32_t i = (uint32_t)lane; i < nw; i += (uint32_t)nthr) {
        uint32_t v;
        if (i == 0 && sh) v = solo_bits32(p, wimg, 0, TB < 32 - sh ? TB : 32 - sh) << sh;
        else v = solo_bits32(p, wimg, 32 * i - sh, TB);
        const bool shared = (i == 0 && sh) || (i == nw - 1 && ((sh + TB) & 31) && !at_end);
        put_bits_word(p, out, w0 + i, v, shared);
    }
}

// stream layout: the group's shared-memory stream already is the packed bits
__device__ void solo_write_stream_bits(const Params &p, const uint32_t *st, long long env0, int nenv, int lane,
                                       int nthr) {
    uint32_t *out = reinterpret_cast<uint32_t *>(p.obs);
    const unsigned long long g0 = (unsigned long long)env0 * p.PE;
    const uint32_t TB = (uint32_t)nenv * p.PE, sh = (uint32_t)(g0 & 31);
    const unsigned long long w0 = g0 >> 5;
    const uint32_t nw = (sh + TB + 31) >> 5, nwl = (TB + 31) >> 5;
    const bool at_end = env0 + nenv >= p.B;
    for (uint32_t i = (uint32_t)lane; i < nw; i += (uint32_t)nthr) {
        uint32_t a = i < nwl ? st[sidx(i)] : 0u;
        if (i == nwl - 1 && (TB & 31)) a &= (1u << (TB & 31)) - 1u;
        uint32_t v = a;
        if (sh) {
            uint32_t b = i >= 1 ? st[sidx(i - 1)] : 0u;
            if (i - 1 == nwl - 1 && (TB & 31)) b &= (1u << (TB & 31)) - 1u;
            v = (a << sh) | (i >= 1 ? (b >> (32 - sh)) : 0u);
        }
        const bool shared = (i == 0 && sh) || (i == nw - 1 && ((sh + TB) & 31) && !at_end);
        put_bits_word(p, out, w0 + i, v, shared);
    }
}

// Block mode (small batches: a warp steps at most a few envs): the warp renders
// each of its envs together -- lane l builds window rows l, l+32, ... of every
// plane and ORs them into the zeroed slot -- instead of one lane streaming the
// whole image bit by bit (the serial render was ~40% of c1's latency).
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_render_coop(const Params &p, const SoloEnv<DOM> &src, int owner, uint32_t *slot,
                                                 int lane) {
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL;
    SB pl[NPL], frz;
#pragma unroll
    for (int k = 0; k < 8; k++) {
#pragma unroll
        for (int q = 0; q < NPL; q++) pl[q].w[k] = __shfl_sync(0xffffffffu, src.pl[q].w[k], owner);
        frz.w[k] = __shfl_sync(0xffffffffu, src.frz.w[k], owner);
    }
    const int h = __shfl_sync(0xffffffffu, src.h, owner), w = __shfl_sync(0xffffffffu, src.w, owner);
    const int pr = __shfl_sync(0xffffffffu, src.pr, owner), pc = __shfl_sync(0xffffffffu, src.pc, owner);
    const int OH = p.OH, OW = p.OW, H = p.H, W = p.W;
    for (int i = lane; i < p.env_smem; i += 32) slot[i] = 0u;  // the slot (elided or not)
    __syncwarp();
    const int r0 = rep_of<S>(p) != REP_WIDE ? pr - p.half : 0, c0 = rep_of<S>(p) != REP_WIDE ? pc - p.half : 0;
    const int jlo = c0 < 0 ? -c0 : 0;
    const int jhi = (W - c0) < OW ? (W - c0) : OW;
    const uint64_t full = OW >= 64 ? ~0ull : ((1ull << OW) - 1ull);
    const uint64_t inside = (jhi > jlo ? (jhi >= 64 ? ~0ull : ((1ull << jhi) - 1ull)) : 0ull) & ~((1ull << jlo) - 1ull);
    const uint32_t wm = mask16(W), am = mask16(w);
    const int planes = N + 2 - p.elide;
    for (int idx = lane; idx < planes * OH; idx += 32) {
        const int pln = idx / OH, i = idx - pln * OH, gr = r0 + i;
        const bool fill = pln >= N;  // border and frozen planes read 1 outside the max grid
        uint64_t win;
        if (gr < 0 || gr >= H) {
            win = fill ? full : 0ull;
        } else {
            const int k = gr >> 1, sh = (gr & 1) * 16;
            uint32_t any = 0, sel = 0, fz = 0;
#pragma unroll
            for (int kk = 0; kk < 8; kk++) {
                if (kk == k) {
#pragma unroll
                    for (int q = 0; q < NPL; q++) {
                        any |= pl[q].w[kk];
                        sel |= pl[q].w[kk] & (0u - (uint32_t)(q == pln - 1));
                    }
                    fz = frz.w[kk];
                }
            }
            any = (any >> sh) & 0xFFFFu;
            sel = (sel >> sh) & 0xFFFFu;
            fz = (fz >> sh) & 0xFFFFu;
            const uint32_t act = gr < h ? am : 0u;
            const uint32_t m = pln == 0 ? (act & ~any) : pln < N ? sel : pln == N ? (~act & wm) : fz;
            win = c0 >= 0 ? ((uint64_t)m >> c0) : ((uint64_t)m << (-c0));
            win = (win & inside) | (fill ? (full & ~inside) : 0ull);
        }
        if (!win) continue;
        const uint32_t off = (uint32_t)pln * p.OO + (uint32_t)i * OW, w0 = off >> 5, bs = off & 31;
        const uint64_t a = win << bs;
        const uint32_t carry = bs ? (uint32_t)(win >> (64 - bs)) : 0u;
        if ((uint32_t)a) atomicOr(slot + w0, (uint32_t)a);
        if ((uint32_t)(a >> 32)) atomicOr(slot + w0 + 1, (uint32_t)(a >> 32));
        if (carry) atomicOr(slot + w0 + 2, carry);
    }
    __syncwarp();
}

// One env, one thread: step / reset / observe (solo_begin + solo_finish), then
// render its image into `slot`. A step's observation depends only on the tiles
// after the action and the next scan position -- not on the metrics -- unless
// the episode ends (auto-reset) or control planes are rendered, so the warp
// can render and start storing before it recomputes (env_solo_body).
template <int DOM>
struct SoloStep {
    SoloEnv<DOM> e;
    bool cold, rows_dirty, planes_dirty, metrics_dirty, rng_dirty, wrote, reset_now, ends;
    double before;
};

// load; apply the action (env.py:355-372); advance the scan position and t
// (env.py:374-381: independent of the recompute)
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_begin(const Params &p, int mode, long long env, SoloStep<DOM> &st) {
    constexpr int N = Dom<DOM>::N;
    SoloEnv<DOM> &e = st.e;
    solo_load_hot<DOM, S>(p, env, e);
    // control planes render the metric values; reset/recompute/reprice use everything
    st.cold = (mode != MODE_STEP && mode != MODE_OBSERVE) || nctrl_of<S>(p) > 0;
    if (st.cold) solo_load_cold<DOM, S>(p, env, e, true);
    st.rows_dirty = st.planes_dirty = st.metrics_dirty = st.rng_dirty = false;
    st.wrote = st.reset_now = st.ends = false;
    st.before = 0.0;
    if (mode == MODE_STEP) {
        long long a = step_action(p, env, true);
        bool ok = a >= 0 && a < p.n_actions;
        if (!ok) atomicOr(p.err, (unsigned)FLAG_BAD_ACTION);
        int r = e.pr, c = e.pc, tile = -1;
        if (rep_of<S>(p) == REP_NARROW) {
            if (ok && a != 0) tile = (int)a - 1;
        } else if (rep_of<S>(p) == REP_TURTLE) {
            if (ok && a < 4) {
                if (a == 0) r = r > 0 ? r - 1 : 0;
                else if (a == 1) r = r < e.h - 1 ? r + 1 : e.h - 1;
                else if (a == 2) c = c > 0 ? c - 1 : 0;
                else c = c < e.w - 1 ? c + 1 : e.w - 1;
                e.pr = r;
                e.pc = c;
            } else if (ok) {
                tile = (int)a - 4;
            }
        } else if (ok) {  // wide
            int cell = (int)(a / N);
            tile = (int)(a - (long long)cell * N);
            r = cell / p.W;
            c = cell - r * p.W;
        }
        if (tile >= 0) {
            const uint32_t sh = (r & 1) * 16 + c;
            const int wi = r >> 1;
            bool act = r < e.h && c < e.w;
            int cur = act ? 0 : N;
            uint32_t fz = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k == wi) {
#pragma unroll
                    for (int q = 0; q < Dom<DOM>::NPL; q++)
                        if ((e.pl[q].w[k] >> sh) & 1u) cur = q + 1;
                    fz = (e.frz.w[k] >> sh) & 1u;
                }
            }
            bool editable = act && !fz;
            st.wrote = tile != cur && (rep_of<S>(p) == REP_NARROW || editable);
        }
        if (st.wrote) {  // env.py:369-372
            solo_set_tile<DOM, S>(e, r, c, tile);
            st.planes_dirty = true;
            e.changes += 1;
        }
        if (rep_of<S>(p) == REP_NARROW) {  // pos_idx = (pos_idx + 1) % order_len
            SB ed = andnot(rect_sb(e.h, e.w), e.frz);
            int nidx = e.pos_idx + 1, nxt;
            if (nidx >= e.order_len) {
                nidx = 0;
                nxt = solo_serp_first(ed, 0);
            } else {
                nxt = solo_serp_next(ed, e.pr, e.pc);
            }
            nxt = max(nxt, 0);  // no editable cell left (imported state): stay well-formed
            e.pos_idx = nidx;
            e.pr = nxt >> 4;
            e.pc = nxt & 15;
        }
        e.t += 1;
        // the episode ends this step (done depends only on counters)
        st.ends = e.t >= e.max_steps || (p.budget > 0 && e.changes >= p.budget);
    } else if (mode == MODE_RESET) {
        st.reset_now = !p.reset_mask || p.reset_mask[env];
    } else if (mode == MODE_RECOMPUTE) {
        st.wrote = !p.reset_mask || p.reset_mask[env];  // recompute without a write
    } else if (mode == MODE_REPRICE) {
        if (!p.reset_mask || p.reset_mask[env]) e.prev_loss = loss_of<DOM>(p, e.val, e.unr, e.lo, e.hi);
    }
}

// recompute (env.py:332-347), reward/done/info (env.py:373-390), auto-reset
// (env.py:391-392), state write-back
template <int DOM, int S = 0>
__device__ __forceinline__ void solo_finish(const Params &p, int mode, long long env, SoloStep<DOM> &st, void *slot) {
    SoloEnv<DOM> &e = st.e;
    if (mode == MODE_STEP) {
        if (!st.cold && (st.wrote || st.ends)) {
            solo_load_cold<DOM, S>(p, env, e, false);
            st.cold = true;
        }
        st.before = e.prev_loss;
    }
    // pass 0: the step's recompute + bookkeeping; pass 1: auto-reset. One
    // call site for the metric code keeps the kernel's instruction footprint small.
#pragma unroll 1
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            if (!st.reset_now) break;
            solo_reset_setup<DOM, S>(p, e);
            st.rows_dirty = true;
        }
        if (pass == 1 || st.wrote) {
            solo_recompute<DOM, S>(p, e, slot, pass == 1);  // _recompute (env.py:332-347)
            st.metrics_dirty = st.rng_dirty = true;
        }
        if (pass == 0 && mode == MODE_STEP) {
            double reward = st.wrote ? __dsub_rn(st.before, e.prev_loss) : 0.0;
            e.ep_reward = __dadd_rn(e.ep_reward, reward);
            const bool done = st.ends;
            p.reward[env] = reward;
            p.done[env] = done;
            if (p.terminal) p.terminal[env] = done;
            if (p.ep_rew) p.ep_rew[env] = done ? e.ep_reward : 0.0;
            if (p.ep_len) p.ep_len[env] = done ? e.t : 0;
            if (p.ep_start) p.ep_start[env] = done ? e.ep_start_loss : 0.0;
            if (p.fin_loss) p.fin_loss[env] = done ? e.prev_loss : 0.0;
            if (done && p.stats) block_stats_add(e.ep_reward, (double)e.t, e.ep_start_loss, e.prev_loss);
            st.reset_now = done && !p.no_auto_reset;
        }
    }
    if (mode != MODE_OBSERVE)
        solo_store<DOM, S>(p, env, e, st.rows_dirty, st.planes_dirty, st.metrics_dirty, st.rng_dirty, st.cold);
}

template <int DOM, int S = 0>
__device__ __forceinline__ void solo_env(const Params &p, int mode, long long env, uint32_t *slot, uint32_t *img,
                                         bool stream, uint32_t bit0, bool last) {
    SoloStep<DOM> st;
    solo_begin<DOM, S>(p, mode, env, st);
    solo_finish<DOM, S>(p, mode, env, st, slot);
    if (p.obs) solo_render<DOM, S>(p, st.e, img, stream, bit0, last);
}

#ifndef LG_EARLY_SPLIT
#define LG_EARLY_SPLIT 4  // eighths of the warp's output stored before the recompute
#endif
#ifndef LG_DUNGEON_EARLY
#define LG_DUNGEON_EARLY 0  // dungeon's warp kernel without the early-observation path (c3: spills)
#endif
#ifndef LG_STREAM_U
#define LG_STREAM_U 2  // 256-bit stores in flight per lane in the warp-stream writer
#endif
#ifndef LG_DUNGEON_SPEC_EARLY
#define LG_DUNGEON_SPEC_EARLY 1  // ... but the specialised one (c3) has the registers for it
#endif
// WARP = 1: the warp-mode kernel (E == blockDim: each warp owns 32 envs);
// WARP = 0: the block-mode kernel (small batches). Two kernels, so neither
// carries the other's code paths (register pressure, instruction footprint).
template <int DOM, int WARP, int S = 0>
__device__ __forceinline__ void env_solo_work(const Params &p, int mode) {
    extern __shared__ __align__(16) uint32_t smem_w[];
    const int E = p.solo_E, T = blockDim.x, tid = threadIdx.x;
    constexpr bool warp_mode = WARP == 1;  // the host launches this kernel only when E == T
    if (gate_closed(p)) return;
    (void)E;
    // warp mode (large batches): warp w owns 32 consecutive envs and writes
    // their outputs; block mode (small batches): E < T envs per block and all
    // T threads write them.
    const int lane = tid & 31, warp = tid >> 5;
    const long long env0 = warp_mode ? (long long)blockIdx.x * T + warp * 32 : (long long)blockIdx.x * E;
    // block mode deals envs round-robin over the warps (env j -> warp j % nw),
    // so a warp steps few envs and their divergent paths serialise less.
    const int nw = T >> 5;
    const int local = warp_mode ? lane : lane * nw + warp;
    const int cap = warp_mode ? 32 : E;
    long long rem = (long long)p.B - env0;
    const int nenv = rem < cap ? (rem > 0 ? (int)rem : 0) : cap;
    const long long env = env0 + local;
    const bool valid = local < nenv && (warp_mode || lane < (E + nw - 1) / nw);
    const int wl = warp_mode ? lane : tid, nthr = warp_mode ? 32 : T;
    uint32_t *grp = smem_w + (warp_mode ? (size_t)warp * (p.stream_mode ? (size_t)p.group_words
                                                                        : (size_t)32 * p.env_smem)
                                        : 0);
    uint32_t *scratch, *img;
    if (p.stream_mode) {
        if (p.obs && valid) grp[sidx(((uint32_t)local * p.PE) >> 5)] = 0u;  // shared boundary words
        if (warp_mode) __syncwarp();
        else __syncthreads();
        // union-find scratch: the env's own interior stream words when they
        // are large enough (written by nobody else before this env renders)
        scratch = p.stream_words == 0 ? grp + sidx((((uint32_t)local * p.PE) >> 5) + 1)
                                      : grp + p.stream_words + (size_t)local * 33;
        img = grp;
    } else {
        scratch = img = grp + (size_t)local * p.env_smem;
    }
    // Early observation (warp mode, float32 planes only): render right after
    // the action, store the first half of the warp's output, recompute, then
    // store the rest -- so a launch does not start with every warp computing
    // and no warp storing (one-wave batches: c3; the shards of a multi-GPU c5).
    // Not when an env of the warp ends this step (auto-reset changes its map).
    if (warp_mode && (DOM != 2 || LG_DUNGEON_EARLY || (S != 0 && LG_DUNGEON_SPEC_EARLY)) && p.early && mode == MODE_STEP &&
        p.obs && nctrl_of<S>(p) == 0 && !obs_u8_of<S>(p) && !obs_bits_of<S>(p) &&
        (p.stream_mode || p.PB == p.PE) &&
        (reinterpret_cast<uintptr_t>(p.obs + (size_t)env0 * p.PE) & 31) == 0) {
        SoloStep<DOM> st;
        if (valid) solo_begin<DOM, S>(p, mode, env, st);
        if (!__any_sync(0xffffffffu, valid && st.ends)) {
            if (valid) solo_render<DOM, S>(p, st.e, img, p.stream_mode != 0, (uint32_t)local * p.PE, local == nenv - 1);
            __syncwarp();
            const uint32_t nv = (uint32_t)nenv * p.PE / 8;
            const uint32_t qm = (uint32_t)((uint64_t)nv * LG_EARLY_SPLIT / 8) & ~127u;  // multiple of nthr * U
            if (p.stream_mode) solo_write_stream<8, LG_STREAM_U>(p, grp, env0, nenv, wl, nthr, 0, qm);
            else solo_write_noctrl<LG_WRITER_U>(p, grp, env0, nenv, wl, nthr, 0, qm);
            if (valid) solo_finish<DOM, S>(p, mode, env, st, scratch);
            if (p.stream_mode) solo_write_stream<8, LG_STREAM_U>(p, grp, env0, nenv, wl, nthr, qm);
            else solo_write_noctrl<LG_WRITER_U>(p, grp, env0, nenv, wl, nthr, qm);
            return;
        }
        if (valid) {
            solo_finish<DOM, S>(p, mode, env, st, scratch);
            solo_render<DOM, S>(p, st.e, img, p.stream_mode != 0, (uint32_t)local * p.PE, local == nenv - 1);
        }
    } else if (!warp_mode && p.obs && !p.stream_mode && nctrl_of<S>(p) == 0 && p.coop) {
        SoloStep<DOM> st;
        if (valid) {
            solo_begin<DOM, S>(p, mode, env, st);
            solo_finish<DOM, S>(p, mode, env, st, scratch);
        }
        // this warp's envs are its lanes 0..k-1 (env local = lane * nw + warp)
        const int mine = __popc(__ballot_sync(0xffffffffu, valid));
        for (int k = 0; k < mine; k++)
            solo_render_coop<DOM, S>(p, st.e, k, grp + (size_t)(k * nw + warp) * p.env_smem, lane);
    } else if (valid) {
        solo_env<DOM, S>(p, mode, env, scratch, img, p.stream_mode != 0, (uint32_t)local * p.PE, local == nenv - 1);
    }
    if (p.stream_mode) {
        if (!p.obs) return;
        if (warp_mode) __syncwarp();
        else __syncthreads();
        if (nenv <= 0) return;
        if (obs_bits_of<S>(p)) {
            solo_write_stream_bits(p, grp, env0, nenv, wl, nthr);
        } else if (obs_u8_of<S>(p)) {
            // env0 is a multiple of 32, so the warp's byte range is 32-byte aligned
            solo_write_stream_u8(p, grp, env0, nenv, wl, nthr);
        } else if ((reinterpret_cast<uintptr_t>(p.obs + (size_t)env0 * p.PE) & 31) == 0) {
            solo_write_stream<8, LG_STREAM_U>(p, grp, env0, nenv, wl, nthr);
        } else {
            solo_write_stream<4, 2>(p, grp, env0, nenv, wl, nthr);
        }
        return;
    }
    img = grp;
    if (!p.obs) return;
    if (warp_mode) __syncwarp();
    else __syncthreads();
    if (nenv <= 0) return;
    if (obs_bits_of<S>(p)) {
        solo_write_bits(p, img, env0, nenv, wl, nthr);
        return;
    }
    const size_t first = (size_t)env0 * p.PE;
    if (obs_u8_of<S>(p)) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(reinterpret_cast<uint8_t *>(p.obs) + first);
        if ((a & 31) == 0) solo_write_u8<32>(p, img, env0, nenv, wl, nthr);
        else if ((a & 15) == 0) solo_write_u8<16>(p, img, env0, nenv, wl, nthr);
        else {
            uint8_t *out = reinterpret_cast<uint8_t *>(p.obs) + first;
            for (uint32_t t = wl; t < (uint32_t)nenv * p.PE; t += nthr) {
                uint32_t e2 = fdiv(p.divPE, t), l2 = t - e2 * p.PE;
                out[t] = (img[e2 * (uint32_t)p.env_smem + (l2 >> 5)] >> (l2 & 31)) & 1u;
            }
        }
        return;
    }
    // obs base is 16-byte aligned (checked on the host) and env0 is a multiple
    // of 8, so every block's output starts 32-byte aligned when the base is.
    if ((reinterpret_cast<uintptr_t>(p.obs + first) & 31) == 0) {
        if (p.PB == p.PE) solo_write_noctrl<LG_WRITER_U>(p, img, env0, nenv, wl, nthr);
        else solo_write<8, 2>(p, img, env0, nenv, wl, nthr);
    } else {
        solo_write<4, 2>(p, img, env0, nenv, wl, nthr);
    }
}

template <int DOM, int WARP, int S = 0>
__device__ __forceinline__ void env_solo_body(const Params &p, int mode) {
    chain_enter(p);
    block_stats_begin(p, mode);
    env_solo_work<DOM, WARP, S>(p, mode);
    block_stats_flush(p, mode);
    chain_leave(p);
}

// Register caps (measured): binary runs 8 x 64-thread blocks per SM at 128
// registers (8 bytes of spills; with the early-observation split it would
// otherwise take 133 and 7 blocks: 131k-env shard 366 M vs 355 M, c5 equal);
// maze/dungeon run faster at 8 blocks (128 regs) despite spills (c3: 418 M
// vs 343 M env-steps/s at 144).
#ifndef LG_BINARY_NREG
#define LG_BINARY_NREG 128
#endif
__global__ void __maxnreg__(LG_BINARY_NREG) env_solo_kernel_binary(const Params p, int mode) { env_solo_body<0, 1>(p, mode); }
__global__ void __maxnreg__(128) env_solo_kernel_maze(const Params p, int mode) { env_solo_body<1, 1>(p, mode); }
__global__ void __maxnreg__(128) env_solo_kernel_dungeon(const Params p, int mode) { env_solo_body<2, 1>(p, mode); }
__global__ void __maxnreg__(128) env_solo_kernel_binary_small(const Params p, int mode) { env_solo_body<0, 0>(p, mode); }
__global__ void __maxnreg__(128) env_solo_kernel_maze_small(const Params p, int mode) { env_solo_body<1, 0>(p, mode); }
__global__ void __maxnreg__(128) env_solo_kernel_dungeon_small(const Params p, int mode) { env_solo_body<2, 0>(p, mode); }
// specialised (env_kernels.cuh spec_of): c5 / c1 (binary narrow, no pins), c3 (dungeon wide)
constexpr int SOLO_SPEC_BINARY = spec_of(REP_NARROW, true), SOLO_SPEC_DUNGEON = spec_of(REP_WIDE, false);
__global__ void __maxnreg__(LG_BINARY_NREG) env_solo_kernel_binary_s(const Params p, int mode) {
    env_solo_body<0, 1, SOLO_SPEC_BINARY>(p, mode);
}
__global__ void __maxnreg__(128) env_solo_kernel_binary_small_s(const Params p, int mode) {
    env_solo_body<0, 0, SOLO_SPEC_BINARY>(p, mode);
}
#ifndef LG_DUNGEON_S_NREG
#define LG_DUNGEON_S_NREG 128
#endif
__global__ void __maxnreg__(LG_DUNGEON_S_NREG) env_solo_kernel_dungeon_s(const Params p, int mode) {
    env_solo_body<2, 1, SOLO_SPEC_DUNGEON>(p, mode);
}

template <int DOM>
struct SoloKernel;
template <>
struct SoloKernel<0> {
    static constexpr auto fn = env_solo_kernel_binary;
    static constexpr auto fn_small = env_solo_kernel_binary_small;
    static constexpr int spec = SOLO_SPEC_BINARY;
    static constexpr auto fn_spec = env_solo_kernel_binary_s;
    static constexpr auto fn_small_spec = env_solo_kernel_binary_small_s;
};
template <>
struct SoloKernel<1> {
    static constexpr auto fn = env_solo_kernel_maze;
    static constexpr auto fn_small = env_solo_kernel_maze_small;
    static constexpr int spec = 0;
    static constexpr auto fn_spec = env_solo_kernel_maze;
    static constexpr auto fn_small_spec = env_solo_kernel_maze_small;
};
template <>
struct SoloKernel<2> {
    static constexpr auto fn = env_solo_kernel_dungeon;
    static constexpr auto fn_small = env_solo_kernel_dungeon_small;
    static constexpr int spec = SOLO_SPEC_DUNGEON;
    static constexpr auto fn_spec = env_solo_kernel_dungeon_s;
    static constexpr auto fn_small_spec = env_solo_kernel_dungeon_small;  // block mode: generic
};

// ---- state export / import / metrics for the solo layout -------------------

template <int DOM>
__global__ void solo_export_kernel(const Params p, lg_state dst) {
    constexpr int N = Dom<DOM>::N, NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    const long long env = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (env >= p.B) return;
    SoloEnv<DOM> e;
    solo_load<DOM>(p, env, e);
    const int H = p.H, W = p.W, HW = H * W;
    SB act = rect_sb(e.h, e.w);
    SB ed = andnot(act, e.frz);
    int32_t *ord = dst.order + (size_t)env * HW;
    int n = 0;
    for (int r = 0; r < H; r++) {
        uint32_t arow = act.row(r), frow = e.frz.row(r), erow = ed.row(r);
        uint32_t prow[NPL];
#pragma unroll
        for (int q = 0; q < NPL; q++) prow[q] = e.pl[q].row(r);
        for (int c = 0; c < W; c++) {
            bool a = (arow >> c) & 1u;
            int tile = a ? 0 : N;
#pragma unroll
            for (int q = 0; q < NPL; q++)
                if ((prow[q] >> c) & 1u) tile = q + 1;
            size_t o = ((size_t)env * H + r) * W + c;
            dst.tiles[o] = (uint8_t)tile;
            dst.active[o] = a;
            dst.frozen[o] = (frow >> c) & 1u;
        }
        for (int k = 0; k < W; k++) {
            int c = (r & 1) ? W - 1 - k : k;
            if ((erow >> c) & 1u) ord[n++] = r * W + c;
        }
    }
    for (int i = n; i < HW; i++) ord[i] = -1;
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
    dst.metric_seeds[env] = p.mseed[env];
    uint64_t *rg = dst.rng + 6 * env;
    rg[0] = (uint64_t)(e.g.s >> 64);
    rg[1] = (uint64_t)e.g.s;
    rg[2] = (uint64_t)(e.g.inc >> 64);
    rg[3] = (uint64_t)e.g.inc;
    rg[4] = e.g.has;
    rg[5] = e.g.u;
}

template <int DOM>
__global__ void solo_import_kernel(const Params p, lg_state src) {
    constexpr int NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    const long long env = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (env >= p.B) return;
    const int H = p.H, W = p.W;
    uint32_t wq[NPL + 1][8];
#pragma unroll
    for (int q = 0; q <= NPL; q++)
#pragma unroll
        for (int k = 0; k < 8; k++) wq[q][k] = 0;
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            size_t o = ((size_t)env * H + r) * W + c;
            int tile = src.tiles[o];
            uint32_t bit = 1u << ((r & 1) * 16 + c);
            bool a = src.active[o] != 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k != (r >> 1)) continue;
#pragma unroll
                for (int q = 0; q < NPL; q++)
                    if (a && tile == q + 1) wq[q][k] |= bit;
                if (src.frozen[o]) wq[NPL][k] |= bit;
            }
        }
#pragma unroll
    for (int q = 0; q <= NPL; q++) {
        uint32_t *rw = solo_plane(p, env, q);
#pragma unroll
        for (int k = 0; k < 8; k++) rw[k] = wq[q][k];
    }
    Hot hv;
    uint32_t h = (uint32_t)src.shape_hw[2 * env], w = (uint32_t)src.shape_hw[2 * env + 1];
    {  // frozen plane != border plane (~active rectangle) inside the max grid?
        const uint32_t wm = mask16(W), am = mask16((int)w);
        uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint32_t g0 = 2 * k < H ? wm : 0u, g1 = 2 * k + 1 < H ? wm : 0u;
            const uint32_t a0 = 2 * k < (int)h ? am : 0u, a1 = 2 * k + 1 < (int)h ? am : 0u;
            const uint32_t border = (g0 & ~a0) | ((g1 & ~a1) << 16);
            diff |= (wq[NPL][k] ^ border) & (g0 | (g1 << 16));
        }
        if (diff && p.aux) atomicOr(p.aux, 1u);
    }
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

// compute_metrics_batch on raw stacks for maps <= 16x16, one grid per thread.
template <int DOM>
__global__ void __launch_bounds__(128) solo_metrics_kernel(long long n, int H, int W, const uint8_t *tiles,
                                                           const uint8_t *active, uint64_t *rng,
                                                           int64_t *values, uint8_t *unreach) {
    extern __shared__ __align__(16) uint32_t smem_w[];
    constexpr int NPL = Dom<DOM>::NPL, M = Dom<DOM>::M;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    void *uf = smem_w + threadIdx.x * 33;
    SB pl[NPL], act = SB::zero();
#pragma unroll
    for (int q = 0; q < NPL; q++) pl[q] = SB::zero();
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            size_t o = ((size_t)b * H + r) * W + c;
            if (!active[o]) continue;
            uint32_t bit = 1u << ((r & 1) * 16 + c);
            int tile = tiles[o];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k != (r >> 1)) continue;
                act.w[k] |= bit;
#pragma unroll
                for (int q = 0; q < NPL; q++)
                    if (tile == q + 1) pl[q].w[k] |= bit;
            }
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
    SoloK k;
    compute_metrics<SoloK, DOM>(k, pl, act, g, uf, val, unr);
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

}  // namespace lg
