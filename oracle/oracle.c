/*
 * oracle.c -- scalar CPU restatement of the reference env step.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/pkg/src/levelgen/.
 *
 * The reference computes distances with a batched max-filter fixpoint
 * (pathfind.py:143-175). Its own scalar definition of the same quantity is
 * the queue BFS bfs_distance (pathfind.py:45-78, strict=False), which is what
 * this file runs per environment; both are pinned equal by the reference's
 * tests (tests/test_pathfind.py:32-67).
 */
#include "oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static _Thread_local char g_err[256];
static char g_err_global[256];
static int g_threads = 0;

const char *or_last_error(void) { return g_err_global; }
void or_set_threads(int n) { g_threads = n; }

static void set_err(const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
#pragma omp critical(or_err)
    snprintf(g_err_global, sizeof g_err_global, "%s", msg);
}

/* ------------------------------------------------------------------------ */
/* numpy random streams (numpy 2.3: bit_generator.pyx SeedSequence,          */
/* pcg64.h, distributions.c). The reference consumes them at env.py:594,303, */
/* grid.py:124-125,186,215 and problems.py:88,154.                          */
/* ------------------------------------------------------------------------ */

typedef struct {
    u128 state, inc;
    int has;
    uint32_t u;
} pcg_t;

#define PCG_MULT (((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL)

static void pcg_load(pcg_t *g, const uint64_t *r) {
    g->state = ((u128)r[0] << 64) | r[1];
    g->inc = ((u128)r[2] << 64) | r[3];
    g->has = (int)r[4];
    g->u = (uint32_t)r[5];
}
static void pcg_store(const pcg_t *g, uint64_t *r) {
    r[0] = (uint64_t)(g->state >> 64);
    r[1] = (uint64_t)g->state;
    r[2] = (uint64_t)(g->inc >> 64);
    r[3] = (uint64_t)g->inc;
    r[4] = (uint64_t)g->has;
    r[5] = g->u;
}
static inline void pcg_step(pcg_t *g) { g->state = g->state * PCG_MULT + g->inc; }
static inline uint64_t pcg_u64(pcg_t *g) {
    pcg_step(g);
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}
static inline uint32_t pcg_u32(pcg_t *g) {
    if (g->has) {
        g->has = 0;
        return g->u;
    }
    uint64_t v = pcg_u64(g);
    g->has = 1;
    g->u = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
static inline double pcg_double(pcg_t *g) {
    return (double)(pcg_u64(g) >> 11) * (1.0 / 9007199254740992.0);
}
/* random_bounded_uint64 with use_masked=False: result in [0, rng]. */
static uint64_t pcg_bounded(pcg_t *g, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFULL) {
        if (rng == 0xFFFFFFFFULL) return pcg_u32(g);
        uint32_t ex = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)pcg_u32(g) * ex;
        uint32_t left = (uint32_t)m;
        if (left < ex) {
            uint32_t th = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % ex;
            while (left < th) {
                m = (uint64_t)pcg_u32(g) * ex;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
    if (rng == 0xFFFFFFFFFFFFFFFFULL) return pcg_u64(g);
    uint64_t ex = rng + 1;
    u128 m = (u128)pcg_u64(g) * ex;
    uint64_t left = (uint64_t)m;
    if (left < ex) {
        uint64_t th = (0xFFFFFFFFFFFFFFFFULL - rng) % ex;
        while (left < th) {
            m = (u128)pcg_u64(g) * ex;
            left = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}
/* Generator.integers(lo, hi) (exclusive hi). */
static int64_t pcg_integers(pcg_t *g, int64_t lo, int64_t hi) {
    return lo + (int64_t)pcg_bounded(g, (uint64_t)(hi - lo - 1));
}
/* Generator.choice(pop, size=k, replace=False): Floyd + bounded shuffle. */
static int pcg_choice_noreplace(pcg_t *g, int64_t pop, int k, int64_t *out) {
    uint64_t mask = (uint64_t)(1.2 * (double)k);
    for (int s = 1; s <= 32; s <<= 1) mask |= mask >> s;
    uint64_t size = mask + 1;
    uint64_t *hs = (uint64_t *)malloc(size * sizeof(uint64_t));
    if (!hs) return -1;
    for (uint64_t i = 0; i < size; i++) hs[i] = ~0ULL;
    for (int64_t j = pop - k; j < pop; j++) {
        uint64_t val = pcg_bounded(g, (uint64_t)j);
        uint64_t loc = val & mask;
        while (hs[loc] != ~0ULL && hs[loc] != val) loc = (loc + 1) & mask;
        if (hs[loc] == ~0ULL) {
            hs[loc] = val;
            out[j - pop + k] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (hs[loc] != ~0ULL) loc = (loc + 1) & mask;
            hs[loc] = (uint64_t)j;
            out[j - pop + k] = j;
        }
    }
    for (int i = k - 1; i > 0; i--) {
        int64_t j = (int64_t)pcg_bounded(g, (uint64_t)i);
        int64_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
    free(hs);
    return 0;
}

/* SeedSequence mixing (numpy bit_generator.pyx). */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static int u32_words(uint64_t v, uint32_t *w) {
    if (v == 0) {
        w[0] = 0;
        return 1;
    }
    int n = 0;
    while (v) {
        w[n++] = (uint32_t)v;
        v >>= 32;
    }
    return n;
}
static void seedseq_pcg(uint64_t entropy, int has_key, uint64_t key, pcg_t *g) {
    uint32_t ent[8];
    int n = u32_words(entropy, ent);
    if (has_key) {
        while (n < 4) ent[n++] = 0;
        n += u32_words(key, ent + n);
    }
    uint32_t hc = SS_INIT_A, pool[4];
#define HASHMIX(v_, out_)            \
    do {                             \
        uint32_t vv = (v_) ^ hc;     \
        hc *= SS_MULT_A;             \
        vv *= hc;                    \
        vv ^= vv >> 16;              \
        (out_) = vv;                 \
    } while (0)
#define MIX(x_, y_) ((((SS_MIX_L * (x_)) - (SS_MIX_R * (y_))) ^ (((SS_MIX_L * (x_)) - (SS_MIX_R * (y_))) >> 16)))
    for (int i = 0; i < 4; i++) HASHMIX(i < n ? ent[i] : 0u, pool[i]);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) {
                uint32_t h;
                HASHMIX(pool[s], h);
                pool[d] = MIX(pool[d], h);
            }
    for (int s = 4; s < n; s++)
        for (int d = 0; d < 4; d++) {
            uint32_t h;
            HASHMIX(ent[s], h);
            pool[d] = MIX(pool[d], h);
        }
    uint32_t hb = SS_INIT_B, w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3] ^ hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    uint64_t s0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    uint64_t s1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    uint64_t s2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
    uint64_t s3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
    u128 initstate = ((u128)s0 << 64) | s1;
    u128 initseq = ((u128)s2 << 64) | s3;
    g->inc = (initseq << 1) | 1;
    g->state = 0;
    pcg_step(g);
    g->state += initstate;
    pcg_step(g);
    g->has = 0;
    g->u = 0;
#undef HASHMIX
#undef MIX
}

int or_seed_streams(uint64_t seed, int64_t offset, int64_t n, uint64_t *rng_out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        pcg_t g;
        seedseq_pcg(seed, 1, (uint64_t)(offset + i), &g);
        pcg_store(&g, rng_out + 6 * i);
    }
    return 0;
}
int or_seed_plain(uint64_t seed, uint64_t *rng_out) {
    pcg_t g;
    seedseq_pcg(seed, 0, 0, &g);
    pcg_store(&g, rng_out);
    return 0;
}

int or_rng_draw(uint64_t *rng, int kind, int64_t arg, int64_t arg2, int64_t n, uint64_t *out) {
    pcg_t g;
    pcg_load(&g, rng);
    for (int64_t i = 0; i < n; i++) {
        switch (kind) {
        case 0: out[i] = pcg_u64(&g); break;
        case 1: out[i] = pcg_u32(&g); break;
        case 2: {
            double d = pcg_double(&g);
            memcpy(&out[i], &d, 8);
        } break;
        case 3: out[i] = (uint64_t)pcg_integers(&g, 0, arg); break;
        case 4: {
            int64_t tmp[64];
            if (arg2 > 64) return -1;
            pcg_choice_noreplace(&g, arg, (int)arg2, tmp);
            for (int k = 0; k < arg2; k++) out[i * arg2 + k] = (uint64_t)tmp[k];
        } break;
        default: return -1;
        }
    }
    pcg_store(&g, rng);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* domain tables (tiles.py:126-171)                                          */
/* ------------------------------------------------------------------------ */

enum { T_AIR = 0, T_WALL = 1 };
/* maze ids */
enum { MZ_PLAYER = 2, MZ_DOOR = 3 };
/* dungeon ids */
enum { DG_ENEMY = 2, DG_KEY = 3, DG_DOOR = 4, DG_PLAYER = 5 };

static int dom_ntiles(int d) { return d == OR_BINARY ? 2 : d == OR_MAZE ? 4 : 6; }
static int dom_nmetrics(int d) { return d == OR_BINARY ? 2 : d == OR_MAZE ? 4 : 7; }
/* metric kinds for default_targets (problems.py:48-62) */
enum { K_MAX = 0, K_ONE = 1, K_NEAREST = 2, K_NENEMY = 3 };
static int metric_kind(int d, int m) {
    if (m == 0) return K_MAX; /* diameter / path_length / pkd_path */
    if (d == OR_DUNGEON && m == 5) return K_NENEMY;
    if (d == OR_DUNGEON && m == 6) return K_NEAREST;
    return K_ONE;
}
static int metric_is_path(int d, int m) {
    if (d == OR_MAZE) return m == 0;
    if (d == OR_DUNGEON) return m == 0 || m == 6;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* grid kernels (pathfind.py)                                                */
/* ------------------------------------------------------------------------ */

/* bfs_distance(strict=False) (pathfind.py:45-78) == flood_distance (86-113). */
static void bfs(int H, int W, const uint8_t *pass, const uint8_t *src, int32_t *dist, int32_t *q) {
    int head = 0, tail = 0;
    for (int i = 0; i < H * W; i++) {
        dist[i] = -1;
    }
    for (int i = 0; i < H * W; i++)
        if (src[i]) {
            dist[i] = 0;
            q[tail++] = i;
        }
    while (head < tail) {
        int c = q[head++];
        int r = c / W, col = c % W, nd = dist[c] + 1;
        int nb[4] = {r > 0 ? c - W : -1, r < H - 1 ? c + W : -1, col > 0 ? c - 1 : -1,
                     col < W - 1 ? c + 1 : -1};
        for (int k = 0; k < 4; k++) {
            int x = nb[k];
            if (x >= 0 && pass[x] && dist[x] == -1) {
                dist[x] = nd;
                q[tail++] = x;
            }
        }
    }
}

/* count_regions (pathfind.py:116-130): number of 4-connected components. */
static int64_t regions(int H, int W, const uint8_t *pass, int32_t *lab, int32_t *q) {
    int64_t n = 0;
    for (int i = 0; i < H * W; i++) lab[i] = 0;
    for (int s = 0; s < H * W; s++) {
        if (!pass[s] || lab[s]) continue;
        n++;
        int head = 0, tail = 0;
        q[tail++] = s;
        lab[s] = 1;
        while (head < tail) {
            int c = q[head++];
            int r = c / W, col = c % W;
            int nb[4] = {r > 0 ? c - W : -1, r < H - 1 ? c + W : -1, col > 0 ? c - 1 : -1,
                         col < W - 1 ? c + 1 : -1};
            for (int k = 0; k < 4; k++) {
                int x = nb[k];
                if (x >= 0 && pass[x] && !lab[x]) {
                    lab[x] = 1;
                    q[tail++] = x;
                }
            }
        }
    }
    return n;
}

/* endpoint_field (pathfind.py:188-203) followed by _masked_min
 * (problems.py:98-102) over `mask`; returns big (= H*W+2) when nothing. */
static int64_t endpoint_min(int H, int W, const int32_t *dist, const uint8_t *mask) {
    int32_t big = H * W + 2;
    int64_t best = big;
    for (int c = 0; c < H * W; c++) {
        if (!mask[c]) continue;
        int32_t d = dist[c] == -1 ? big : dist[c];
        int r = c / W, col = c % W;
        int32_t via = big;
        int nb[4] = {r > 0 ? c - W : -1, r < H - 1 ? c + W : -1, col > 0 ? c - 1 : -1,
                     col < W - 1 ? c + 1 : -1};
        for (int k = 0; k < 4; k++) {
            int x = nb[k];
            if (x >= 0) {
                int32_t dx = dist[x] == -1 ? big : dist[x];
                if (dx < via) via = dx;
            }
        }
        via += 1;
        int32_t o = d < via ? d : via;
        if (o >= big) continue; /* UNREACHABLE */
        if (o < best) best = o;
    }
    return best;
}
/* _masked_min over raw distances (problems.py:98-102). */
static int64_t raw_min(int H, int W, const int32_t *dist, const uint8_t *mask) {
    int64_t best = H * W + 2;
    for (int c = 0; c < H * W; c++)
        if (mask[c] && dist[c] != -1 && dist[c] < best) best = dist[c];
    return best;
}

typedef struct {
    uint8_t *pass, *src, *m1, *m2, *m3;
    int32_t *dist, *dist2, *q;
} scratch_t;

static int scratch_init(scratch_t *s, int HW) {
    s->pass = (uint8_t *)malloc(5 * (size_t)HW);
    s->dist = (int32_t *)malloc(3 * (size_t)HW * sizeof(int32_t));
    if (!s->pass || !s->dist) return -1;
    s->src = s->pass + HW;
    s->m1 = s->src + HW;
    s->m2 = s->m1 + HW;
    s->m3 = s->m2 + HW;
    s->dist2 = s->dist + HW;
    s->q = s->dist2 + HW;
    return 0;
}
static void scratch_free(scratch_t *s) {
    free(s->pass);
    free(s->dist);
}

/* compute_metrics_batch for one grid (problems.py:105-243).
 * `g` is the metric generator (binary only). */
static void metrics_one(int domain, int H, int W, const uint8_t *tiles, const uint8_t *active,
                        pcg_t *g, int64_t *val, uint8_t *unr, scratch_t *s) {
    int HW = H * W;
    int32_t big = HW + 2;
    int M = dom_nmetrics(domain);
    for (int m = 0; m < M; m++) {
        val[m] = 0;
        unr[m] = 0;
    }
    if (domain == OR_BINARY) {
        /* _binary_metrics (problems.py:136-173) */
        int64_t count = 0;
        for (int i = 0; i < HW; i++) {
            s->pass[i] = (uint8_t)(tiles[i] == T_AIR && active[i]);
            count += s->pass[i];
        }
        val[1] = regions(H, W, s->pass, s->dist2, s->q);
        if (count > 0) {
            int64_t k = pcg_integers(g, 0, count);
            int start = -1;
            for (int i = 0; i < HW; i++)
                if (s->pass[i] && k-- == 0) {
                    start = i;
                    break;
                }
            memset(s->src, 0, HW);
            s->src[start] = 1;
            bfs(H, W, s->pass, s->src, s->dist, s->q);
            int y = 0;
            for (int i = 1; i < HW; i++)
                if (s->dist[i] > s->dist[y]) y = i; /* np.argmax: first max */
            memset(s->src, 0, HW);
            s->src[y] = 1;
            bfs(H, W, s->pass, s->src, s->dist, s->q);
            int32_t mx = -1;
            for (int i = 0; i < HW; i++)
                if (s->dist[i] > mx) mx = s->dist[i];
            val[0] = mx;
        }
        return;
    }
    if (domain == OR_MAZE) {
        /* _maze_metrics (problems.py:176-198) */
        int64_t np_ = 0, nd = 0;
        for (int i = 0; i < HW; i++) {
            uint8_t t = tiles[i], a = active[i];
            s->pass[i] = (uint8_t)(a && (t == T_AIR || t == MZ_PLAYER || t == MZ_DOOR));
            s->src[i] = (uint8_t)(a && t == MZ_PLAYER);
            s->m1[i] = (uint8_t)(a && t == MZ_DOOR);
            np_ += s->src[i];
            nd += s->m1[i];
        }
        val[2] = np_;
        val[3] = nd;
        val[1] = regions(H, W, s->pass, s->dist2, s->q);
        bfs(H, W, s->pass, s->src, s->dist, s->q);
        int64_t best = raw_min(H, W, s->dist, s->m1);
        int bad = np_ == 0 || nd == 0 || best >= big;
        val[0] = bad ? 0 : best;
        unr[0] = (uint8_t)bad;
        return;
    }
    /* _dungeon_metrics (problems.py:201-243) */
    int64_t cp = 0, ck = 0, cd = 0, ce = 0;
    for (int i = 0; i < HW; i++) {
        uint8_t t = tiles[i], a = active[i];
        s->pass[i] = (uint8_t)(a && (t == T_AIR || t == DG_PLAYER));
        s->src[i] = (uint8_t)(a && t == DG_PLAYER);
        s->m1[i] = (uint8_t)(a && t == DG_KEY);
        s->m2[i] = (uint8_t)(a && t == DG_DOOR);
        s->m3[i] = (uint8_t)(a && t == DG_ENEMY);
        cp += s->src[i];
        ck += s->m1[i];
        cd += s->m2[i];
        ce += s->m3[i];
    }
    val[2] = cp;
    val[3] = ck;
    val[4] = cd;
    val[5] = ce;
    bfs(H, W, s->pass, s->src, s->dist, s->q); /* from players */
    int64_t leg1 = endpoint_min(H, W, s->dist, s->m1);
    int64_t near = endpoint_min(H, W, s->dist, s->m3);
    bfs(H, W, s->pass, s->m1, s->dist, s->q); /* from keys */
    int64_t leg2 = endpoint_min(H, W, s->dist, s->m2);
    int missing = cp == 0 || ck == 0 || cd == 0;
    int bad = missing || leg1 >= big || leg2 >= big;
    val[0] = bad ? 0 : leg1 + leg2;
    unr[0] = (uint8_t)bad;
    int badn = cp == 0 || ce == 0 || near >= big;
    val[6] = badn ? 0 : near;
    unr[6] = (uint8_t)badn;
    /* regions over {AIR, PLAYER, KEY, DOOR} */
    for (int i = 0; i < HW; i++) {
        uint8_t t = tiles[i];
        s->pass[i] = (uint8_t)(active[i] && (t == T_AIR || t == DG_PLAYER || t == DG_KEY || t == DG_DOOR));
    }
    val[1] = regions(H, W, s->pass, s->dist2, s->q);
}

int or_metrics(int domain, int H, int W, int64_t B, const uint8_t *tiles, const uint8_t *active,
               uint64_t *rng, int64_t *values, uint8_t *unreach) {
    int M = dom_nmetrics(domain);
    int err = 0;
#pragma omp parallel
    {
        scratch_t s;
        int ok = scratch_init(&s, H * W) == 0;
        if (!ok) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 64)
        for (int64_t b = 0; b < B; b++) {
            if (!ok) continue;
            int64_t v[8];
            uint8_t u[8];
            pcg_t g;
            memset(&g, 0, sizeof g);
            if (rng) pcg_load(&g, rng + 6 * b);
            metrics_one(domain, H, W, tiles + b * H * W, active + b * H * W, &g, v, u, &s);
            if (rng) pcg_store(&g, rng + 6 * b);
            for (int m = 0; m < M; m++) {
                values[m * B + b] = v[m];
                unreach[m * B + b] = u[m];
            }
        }
        scratch_free(&s);
    }
    return err ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* env (env.py)                                                              */
/* ------------------------------------------------------------------------ */

/* loss_batch (problems.py:251-279): canonical-order float64 accumulation. */
static double loss_of(const or_cfg *cfg, const int64_t *v, const uint8_t *u, const int64_t *lo,
                      const int64_t *hi) {
    int d = cfg->domain, M = dom_nmetrics(d);
    double wreg = cfg->weights[1];
    double total = 0.0;
    for (int m = 0; m < M; m++) {
        double wm = cfg->weights[m];
        double x = (double)v[m], l = (double)lo[m], h = (double)hi[m];
        double a = l - x;
        double b = x - h;
        a = a > 0.0 ? a : 0.0; /* np.maximum(0.0, .) */
        b = b > 0.0 ? b : 0.0;
        double term = wm * (a + b);
        if (metric_is_path(d, m) && u[m]) term = wm * h + wreg;
        total = m == 0 ? term : total + term;
    }
    return total;
}

/* _serpentine_template / scan_order (env.py:155-178). */
static int scan_order(int H, int W, const uint8_t *active, const uint8_t *frozen, int32_t *order) {
    int n = 0;
    for (int r = 0; r < H; r++)
        for (int k = 0; k < W; k++) {
            int c = (r & 1) ? W - 1 - k : k;
            int i = r * W + c;
            if (active[i] && !frozen[i]) order[n++] = i;
        }
    return n;
}

typedef struct {
    const or_cfg *cfg;
    or_state *st;
    int64_t B;
    int H, W, M, n;
} envctx;

static void row_metrics(envctx *e, int64_t b, pcg_t *g, scratch_t *s) {
    int HW = e->H * e->W;
    int64_t v[8];
    uint8_t u[8];
    pcg_t tmp;
    pcg_t *mg = g;
    if (e->cfg->det_metrics) { /* _metric_rngs (env.py:327-330) */
        seedseq_pcg((uint64_t)e->st->metric_seeds[b], 0, 0, &tmp);
        mg = &tmp;
    }
    metrics_one(e->cfg->domain, e->H, e->W, e->st->tiles + b * HW, e->st->active + b * HW, mg, v, u, s);
    for (int m = 0; m < e->M; m++) {
        e->st->values[m * e->B + b] = v[m];
        e->st->unreach[m * e->B + b] = u[m];
    }
}

/* _recompute (env.py:332-347) for one row. */
static double row_recompute(envctx *e, int64_t b, pcg_t *g, scratch_t *s, int reset) {
    row_metrics(e, b, g, s);
    int64_t v[8], lo[8], hi[8];
    uint8_t u[8];
    for (int m = 0; m < e->M; m++) {
        v[m] = e->st->values[m * e->B + b];
        u[m] = e->st->unreach[m * e->B + b];
        lo[m] = e->st->lo[m * e->B + b];
        hi[m] = e->st->hi[m * e->B + b];
    }
    double l = loss_of(e->cfg, v, u, lo, hi);
    e->st->prev_loss[b] = l;
    if (reset) {
        e->st->ep_reward[b] = 0.0;
        e->st->ep_start_loss[b] = l;
    }
    return l;
}

/* reset_rows (env.py:284-305) for one row, incl. _install_row (307-325). */
static int row_reset(envctx *e, int64_t b, scratch_t *s) {
    const or_cfg *cfg = e->cfg;
    or_state *st = e->st;
    int H = e->H, W = e->W, HW = H * W, n = e->n;
    pcg_t g;
    pcg_load(&g, st->rng + 6 * b);
    int h = H, w = W;
    if (cfg->randomize_shape) { /* sample_shape (grid.py:116-126): width then height */
        w = (int)pcg_integers(&g, 3, W + 1);
        h = (int)pcg_integers(&g, 3, H + 1);
    }
    uint8_t *tl = st->tiles + b * HW, *ac = st->active + b * HW, *fr = st->frozen + b * HW;
    /* new_grid + apply_shape (grid.py:105-142) */
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            int a = r < h && c < w;
            ac[r * W + c] = (uint8_t)a;
            fr[r * W + c] = (uint8_t)!a;
            tl[r * W + c] = (uint8_t)(a ? T_AIR : n);
        }
    if (cfg->init_weighted) { /* init_random (grid.py:169-191): choice over the bbox */
        for (int r = 0; r < h; r++)
            for (int c = 0; c < w; c++) {
                double u = pcg_double(&g);
                int idx = 0;
                while (idx < n && cfg->init_cdf[idx] <= u) idx++; /* searchsorted right */
                tl[r * W + c] = (uint8_t)idx;
            }
    } /* else init_empty (grid.py:145-150): already air */
    if (cfg->n_pins > 0) { /* place_pinpoints (grid.py:194-225) */
        int32_t *flat = s->q;
        int nf = 0;
        for (int i = 0; i < HW; i++)
            if (ac[i] && !fr[i]) flat[nf++] = i;
        if (nf < cfg->n_pins) {
            set_err("pinpoints requested but not enough free cells");
            return -1;
        }
        int64_t picks[16];
        pcg_choice_noreplace(&g, nf, cfg->n_pins, picks);
        for (int k = 0; k < cfg->n_pins; k++) {
            int cell = flat[picks[k]];
            tl[cell] = (uint8_t)cfg->pins[k];
            fr[cell] = 1;
        }
    }
    /* sample_control_targets (problems.py:69-90) over default_targets (48-62) */
    int64_t cap = (int64_t)h * w;
    for (int m = 0; m < e->M; m++) {
        int k = metric_kind(cfg->domain, m);
        int64_t lo = 1, hi = 1;
        if (k == K_MAX) lo = hi = cap;
        else if (k == K_NEAREST) {
            lo = 4;
            hi = cap;
        } else if (k == K_NENEMY) {
            lo = 2;
            hi = 5;
        }
        for (int j = 0; j < cfg->n_ctrl; j++)
            if (cfg->ctrl[j] == m) {
                lo = hi = pcg_integers(&g, 0, cap + 1);
            }
        st->lo[m * e->B + b] = lo;
        st->hi[m * e->B + b] = hi;
    }
    /* env.py:302-303: integers(0, 2**63) */
    if (cfg->det_metrics) st->metric_seeds[b] = (int64_t)pcg_bounded(&g, 0x7FFFFFFFFFFFFFFFULL);
    /* _install_row */
    st->shape_hw[2 * b] = h;
    st->shape_hw[2 * b + 1] = w;
    int32_t *ord = st->order + b * HW;
    for (int i = 0; i < HW; i++) ord[i] = -1;
    int len = scan_order(H, W, ac, fr, ord);
    if (len == 0) {
        set_err("no editable cells: every active cell is frozen");
        return -1;
    }
    st->order_len[b] = len;
    st->pos_idx[b] = 0;
    st->pos[2 * b] = ord[0] / W;
    st->pos[2 * b + 1] = ord[0] % W;
    st->t[b] = 0;
    st->changes[b] = 0;
    st->max_steps[b] = cfg->max_steps > 0 ? cfg->max_steps : 3 * cap;
    row_recompute(e, b, &g, s, 1);
    pcg_store(&g, st->rng + 6 * b);
    return 0;
}

static int n_actions(const or_cfg *cfg) {
    int n = dom_ntiles(cfg->domain);
    if (cfg->representation == OR_TURTLE) return 4 + n;
    if (cfg->representation == OR_WIDE) return cfg->max_h * cfg->max_w * n;
    return n + 1;
}

static void ctx_init(envctx *e, const or_cfg *cfg, or_state *st, int64_t B) {
    e->cfg = cfg;
    e->st = st;
    e->B = B;
    e->H = cfg->max_h;
    e->W = cfg->max_w;
    e->M = dom_nmetrics(cfg->domain);
    e->n = dom_ntiles(cfg->domain);
}

#define OMP_THREADS_CLAUSE num_threads(g_threads > 0 ? g_threads : omp_get_max_threads())
#ifndef _OPENMP
static int omp_get_max_threads(void) { return 1; }
#endif

int or_reset(const or_cfg *cfg, or_state *st, int64_t B, const uint8_t *mask) {
    envctx e;
    ctx_init(&e, cfg, st, B);
    int err = 0;
#pragma omp parallel OMP_THREADS_CLAUSE
    {
        scratch_t s;
        if (scratch_init(&s, e.H * e.W)) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 64)
        for (int64_t b = 0; b < B; b++) {
            if (err) continue;
            if (mask && !mask[b]) continue;
            if (row_reset(&e, b, &s)) {
#pragma omp atomic write
                err = 1;
            }
        }
        scratch_free(&s);
    }
    return err ? -1 : 0;
}

int or_step(const or_cfg *cfg, or_state *st, int64_t B, const int64_t *actions, double *reward,
            uint8_t *done, uint8_t *terminal, double *ep_reward, int64_t *ep_length,
            double *ep_start_loss, double *final_loss, int auto_reset) {
    envctx e;
    ctx_init(&e, cfg, st, B);
    int64_t na = n_actions(cfg);
    /* validation before any mutation (env.py:358-361) */
    for (int64_t b = 0; b < B; b++)
        if (actions[b] < 0 || actions[b] >= na) {
            set_err("action id out of range");
            return -1;
        }
    int err = 0;
    int H = e.H, W = e.W, HW = H * W, n = e.n;
#pragma omp parallel OMP_THREADS_CLAUSE
    {
        scratch_t s;
        if (scratch_init(&s, HW)) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 64)
        for (int64_t b = 0; b < B; b++) {
            if (err) continue;
            uint8_t *tl = st->tiles + b * HW, *fr = st->frozen + b * HW, *ac = st->active + b * HW;
            int64_t a = actions[b];
            int r, c, wrote = 0, tile = 0;
            if (cfg->representation == OR_NARROW) { /* env.py:364-372 */
                int flat = st->order[b * HW + st->pos_idx[b]];
                r = flat / W;
                c = flat % W;
                tile = (int)a - 1;
                wrote = a != 0 && tile != tl[flat];
            } else if (cfg->representation == OR_TURTLE) { /* DESIGN.md turtle */
                r = (int)st->pos[2 * b];
                c = (int)st->pos[2 * b + 1];
                if (a < 4) {
                    int h = (int)st->shape_hw[2 * b], w = (int)st->shape_hw[2 * b + 1];
                    if (a == 0) r = r > 0 ? r - 1 : 0;
                    else if (a == 1) r = r < h - 1 ? r + 1 : h - 1;
                    else if (a == 2) c = c > 0 ? c - 1 : 0;
                    else c = c < w - 1 ? c + 1 : w - 1;
                    st->pos[2 * b] = r;
                    st->pos[2 * b + 1] = c;
                } else {
                    tile = (int)a - 4;
                    int i = r * W + c;
                    wrote = ac[i] && !fr[i] && tile != tl[i];
                }
            } else { /* wide: DESIGN.md */
                int64_t cell = a / n;
                tile = (int)(a % n);
                r = (int)(cell / W);
                c = (int)(cell % W);
                int i = r * W + c;
                wrote = ac[i] && !fr[i] && tile != tl[i];
            }
            double rew = 0.0;
            pcg_t g;
            pcg_load(&g, st->rng + 6 * b);
            if (wrote) {
                tl[r * W + c] = (uint8_t)tile;
                st->changes[b] += 1;
                double before = st->prev_loss[b];
                double after = row_recompute(&e, b, &g, &s, 0);
                rew = before - after;
            }
            pcg_store(&g, st->rng + 6 * b);
            st->ep_reward[b] += rew;
            reward[b] = rew;
            if (cfg->representation == OR_NARROW) st->pos_idx[b] = (st->pos_idx[b] + 1) % st->order_len[b];
            if (cfg->representation == OR_NARROW) {
                int flat = st->order[b * HW + st->pos_idx[b]];
                st->pos[2 * b] = flat / W;
                st->pos[2 * b + 1] = flat % W;
            }
            st->t[b] += 1;
            int d = st->t[b] >= st->max_steps[b];
            if (cfg->change_budget > 0) d |= st->changes[b] >= cfg->change_budget;
            done[b] = (uint8_t)d;
            terminal[b] = (uint8_t)d;
            ep_reward[b] = d ? st->ep_reward[b] : 0.0;
            ep_length[b] = d ? st->t[b] : 0;
            ep_start_loss[b] = d ? st->ep_start_loss[b] : 0.0;
            final_loss[b] = d ? st->prev_loss[b] : 0.0;
            if (d && auto_reset) {
                if (row_reset(&e, b, &s)) {
#pragma omp atomic write
                    err = 1;
                }
            }
        }
        scratch_free(&s);
    }
    return err ? -1 : 0;
}

/* build_observation (env.py:186-233); wide uses the whole max grid. */
int or_observe(const or_cfg *cfg, const or_state *st, int64_t B, float *obs) {
    int H = cfg->max_h, W = cfg->max_w, HW = H * W;
    int n = dom_ntiles(cfg->domain), M = dom_nmetrics(cfg->domain);
    int OH, OW;
    if (cfg->representation == OR_WIDE) {
        OH = H;
        OW = W;
    } else {
        OH = OW = cfg->obs_size;
    }
    int C = n + 2 + cfg->n_ctrl;
    int64_t per = (int64_t)C * OH * OW;
#pragma omp parallel for schedule(static) OMP_THREADS_CLAUSE
    for (int64_t b = 0; b < B; b++) {
        float *o = obs + b * per;
        int r0 = 0, c0 = 0;
        if (cfg->representation != OR_WIDE) {
            int half = (cfg->obs_size - 1) / 2;
            r0 = (int)st->pos[2 * b] - half;
            c0 = (int)st->pos[2 * b + 1] - half;
        }
        const uint8_t *tl = st->tiles + b * HW, *fr = st->frozen + b * HW;
        for (int i = 0; i < OH; i++)
            for (int j = 0; j < OW; j++) {
                int r = r0 + i, c = c0 + j;
                int valid = r >= 0 && r < H && c >= 0 && c < W;
                int t = valid ? tl[r * W + c] : n;
                int f = valid ? fr[r * W + c] : 1;
                for (int p = 0; p <= n; p++) o[((int64_t)p * OH + i) * OW + j] = p == t ? 1.0f : 0.0f;
                o[((int64_t)(n + 1) * OH + i) * OW + j] = f ? 1.0f : 0.0f;
            }
        double cap = (double)(st->shape_hw[2 * b] * st->shape_hw[2 * b + 1]);
        for (int k = 0; k < cfg->n_ctrl; k++) {
            int m = cfg->ctrl[k];
            double tgt = ((double)st->lo[m * B + b] + (double)st->hi[m * B + b]) / 2.0;
            double v = ((double)st->values[m * B + b] - tgt) / cap;
            float fv = (float)v;
            float *pl = o + (int64_t)(n + 2 + k) * OH * OW;
            for (int x = 0; x < OH * OW; x++) pl[x] = fv;
        }
    }
    (void)M;
    return 0;
}
