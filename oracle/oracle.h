/*
 * oracle.h -- CPU restatement of the reference env step (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for the CUDA product path. It restates,
 * in plain scalar C, what the reference `levelgen` package computes for the
 * batched PCGRL env step (reference: /root/reference/pkg/src/levelgen/
 * env.py, grid.py, problems.py, pathfind.py, tiles.py), plus the numpy
 * random-stream algorithms the reference consumes (numpy 2.3 SeedSequence,
 * PCG64, Generator.integers/random/choice).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this library against
 * fixtures generated from the live reference (tests/golden/make_golden.py)
 * and against the SURVEY.md Appendix C digests.
 */
#ifndef LG_ORACLE_H
#define LG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_BINARY = 0, OR_MAZE = 1, OR_DUNGEON = 2 };
enum { OR_NARROW = 0, OR_TURTLE = 1, OR_WIDE = 2 };

typedef struct {
    int32_t domain;
    int32_t representation;
    int32_t max_h, max_w;
    int32_t obs_size;
    int32_t randomize_shape;
    int32_t init_weighted;
    int32_t n_pins;
    int32_t pins[16];
    int32_t n_ctrl;
    int32_t ctrl[8];         /* metric indices, canonical order */
    int64_t max_steps;       /* 0 -> 3 * episode area */
    int64_t change_budget;   /* 0 -> unlimited */
    int32_t det_metrics;
    int32_t _pad;
    double init_cdf[8];      /* numpy choice cdf over n_tiles */
    double weights[8];       /* loss weight per metric, canonical order */
} or_cfg;

/* Caller-owned state buffers; layout matches BatchEnv.state_dict()
 * (reference env.py:535-559). [M][B] for lo/hi/values/unreach. */
typedef struct {
    uint8_t *tiles, *active, *frozen;  /* [B][H][W] */
    int64_t *shape_hw;                 /* [B][2] (h, w) */
    int32_t *order;                    /* [B][H*W] */
    int64_t *order_len, *pos_idx;      /* [B] */
    int64_t *pos;                      /* [B][2] current (row, col) (turtle) */
    int64_t *t, *changes, *max_steps;  /* [B] */
    int64_t *lo, *hi, *values;         /* [M][B] */
    uint8_t *unreach;                  /* [M][B] */
    double *prev_loss, *ep_reward, *ep_start_loss; /* [B] */
    int64_t *metric_seeds;             /* [B] */
    uint64_t *rng;                     /* [B][6]: s_hi s_lo inc_hi inc_lo has_u32 uinteger */
} or_state;

const char *or_last_error(void);
void or_set_threads(int n);

/* SeedSequence(seed).spawn(offset+n)[offset+i] -> PCG64 state (env.py:591-594). */
int or_seed_streams(uint64_t seed, int64_t offset, int64_t n, uint64_t *rng_out);
/* default_rng(seed) (no spawn key) -> PCG64 state. */
int or_seed_plain(uint64_t seed, uint64_t *rng_out);

/* _Core.reset_rows (env.py:284-305). mask==NULL resets every row. */
int or_reset(const or_cfg *cfg, or_state *st, int64_t B, const uint8_t *mask);
/* _Core.step (env.py:355-393) + info; auto_reset as BatchEnv.step. */
int or_step(const or_cfg *cfg, or_state *st, int64_t B, const int64_t *actions,
            double *reward, uint8_t *done, uint8_t *terminal, double *ep_reward,
            int64_t *ep_length, double *ep_start_loss, double *final_loss,
            int auto_reset);
/* build_observation (env.py:186-233); wide: full-map window. */
int or_observe(const or_cfg *cfg, const or_state *st, int64_t B, float *obs);

/* compute_metrics_batch (problems.py:105-243) on [B][H][W] stacks.
 * rng: [B][6] streams advanced in place (binary), may be NULL for maze/dungeon. */
int or_metrics(int domain, int H, int W, int64_t B, const uint8_t *tiles,
               const uint8_t *active, uint64_t *rng, int64_t *values, uint8_t *unreach);

/* Raw numpy Generator draws for RNG unit tests. kind: 0 next_u64, 1 next_u32,
 * 2 random() bits as u64, 3 integers(0, arg), 4 choice(arg, k=arg2, replace=False). */
int or_rng_draw(uint64_t *rng, int kind, int64_t arg, int64_t arg2, int64_t n, uint64_t *out);

#ifdef __cplusplus
}
#endif
#endif
