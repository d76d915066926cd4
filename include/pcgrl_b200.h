/*
 * pcgrl_b200.h -- C ABI of the B200-native batched PCGRL env step.
 *
 * Drop-in boundary for the reference's batched environment
 * (levelgen/env.py:486-588, class BatchEnv). The reference is pure Python,
 * so its "FFI" is the Python call surface; each entry point below replaces
 * one reference call (cited per function). The Python host mirror
 * (paper_2408_12525_b200/env.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch types.
 *  - *_dev pointers are caller-owned CUDA device buffers on the env's device;
 *    *_host pointers are host memory (pinned for full copy bandwidth).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All device calls are stream-ordered and asynchronous unless noted.
 *  - return 0 on success, LG_EINVAL (the reference raises ValueError) or
 *    LG_ECUDA (CUDA/runtime failure); lg_last_error() has the message.
 *  - action ids out of range are flagged on device (LG_FLAG_BAD_ACTION) and
 *    the offending env takes a no-op step; lg_errors() reads and clears the
 *    flags (one sync). The reference validates synchronously before mutation
 *    (env.py:358-361); the Python mirror keeps that behaviour for host
 *    actions and with validate=True.
 */
#ifndef PCGRL_B200_H
#define PCGRL_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LG_OK 0
#define LG_EINVAL 1
#define LG_ECUDA 2

#define LG_FLAG_BAD_ACTION 1u      /* env.py:360-361 "action id out of range" */
#define LG_FLAG_NO_EDITABLE 2u     /* env.py:315-316 "no editable cells" */
#define LG_FLAG_PINPOINTS 4u       /* grid.py:213-214 not enough free cells */

enum { LG_BINARY = 0, LG_MAZE = 1, LG_DUNGEON = 2 };
enum { LG_NARROW = 0, LG_TURTLE = 1, LG_WIDE = 2 };
/* Observation buffers are float32 [B][C][OH][OW] as in the reference
 * (env.py:186-233); LG_OBS_U8 writes the same 0/1 planes as uint8 (4x fewer
 * bytes for GPU-side consumers; configs without control planes only);
 * LG_OBS_BITS writes them as one packed stream of ceil(B*C*OH*OW/32) uint32
 * words, element t = bit t%32 of word t/32 (32x fewer bytes; the input of
 * lg_conv1_bits and of the host expansion in lg_step_host). */
enum { LG_OBS_F32 = 0, LG_OBS_U8 = 1, LG_OBS_BITS = 2 };

/* EnvConfig (env.py:42-124) flattened; built by the Python mirror. */
typedef struct {
    int32_t domain;          /* LG_BINARY | LG_MAZE | LG_DUNGEON */
    int32_t representation;  /* LG_NARROW | LG_TURTLE | LG_WIDE */
    int32_t max_h, max_w;    /* 3..64 */
    int32_t obs_size;        /* 3..128 (ignored by wide) */
    int32_t randomize_shape;
    int32_t init_weighted;   /* 1: grid.init_random, 0: grid.init_empty */
    int32_t n_pins;          /* <= 16 */
    int32_t pins[16];        /* pinned tile ids, spec order */
    int32_t n_ctrl;          /* <= 7 */
    int32_t ctrl[8];         /* controllable metric indices, canonical order */
    int64_t max_steps;       /* 0: 3 * episode area */
    int64_t change_budget;   /* 0: unlimited */
    int32_t det_metrics;     /* deterministic_metrics */
    int32_t obs_format;      /* LG_OBS_F32 (reference) | LG_OBS_U8 (opt-in, no controls) */
    double init_cdf[8];      /* numpy choice cdf over the writable tiles */
    double weights[8];       /* loss weight per metric, canonical order */
} lg_config;

/* info dict of BatchEnv.step (env.py:384-390); any pointer may be NULL. */
typedef struct {
    uint8_t *terminal;
    double *episode_reward;
    int64_t *episode_length;
    double *episode_start_loss;
    double *final_loss;
} lg_info;

/* BatchEnv.state_dict() layout (env.py:535-559), all device (or host for
 * the *_host calls) buffers; [M][B] for lo/hi/values/unreach, rng [B][6] =
 * (state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger). */
typedef struct {
    uint8_t *tiles, *active, *frozen;  /* [B][H][W] */
    int64_t *shape_hw;                 /* [B][2] */
    int32_t *order;                    /* [B][H*W], -1 padded */
    int64_t *order_len, *pos_idx;      /* [B] */
    int64_t *pos;                      /* [B][2] current cell (row, col) */
    int64_t *t, *changes, *max_steps;  /* [B] */
    int64_t *lo, *hi, *values;         /* [M][B] */
    uint8_t *unreach;                  /* [M][B] */
    double *prev_loss, *ep_reward, *ep_start_loss; /* [B] */
    int64_t *metric_seeds;             /* [B] */
    uint64_t *rng;                     /* [B][6] */
} lg_state;

typedef struct {
    int64_t n_envs;
    int32_t n_actions;
    int32_t n_metrics;
    int32_t obs_c, obs_h, obs_w;       /* observation_shape (env.py:512-514) */
    int32_t team;                      /* lanes per env in the step kernel */
    int64_t obs_bytes_per_env;
    int64_t state_bytes_per_env;
} lg_desc;

typedef struct lg_env lg_env;

const char *lg_last_error(void);
const char *lg_version(void);

/* BatchEnv.__init__ (env.py:494-497): allocates device state for n_envs
 * environments whose streams are SeedSequence(seed).spawn(...)[global_offset+i]
 * (spawn_rngs, env.py:591-594), so a shard of a multi-GPU batch reproduces
 * the same per-env trajectories as the unsharded batch. */
int lg_create(const lg_config *cfg, int64_t n_envs, int64_t global_offset, uint64_t seed,
              int device, lg_env **out);
int lg_destroy(lg_env *env);
int lg_describe(const lg_env *env, lg_desc *out);

/* BatchEnv.reset (env.py:516-519). obs_dev may be NULL. */
int lg_reset(lg_env *env, void *obs_dev, void *stream);
/* _Core.reset_rows on a subset: mask_dev[b] != 0 resets env b (env.py:284-305). */
int lg_reset_masked(lg_env *env, const uint8_t *mask_dev, void *obs_dev, void *stream);
/* BatchEnv.step (env.py:521-525): actions_dev int64[B]; obs_dev [B,C,OH,OW]
 * (may be NULL to skip the observation), reward_dev f64[B], done_dev u8[B];
 * info may be NULL; stats_dev (NULL or f64[5]) accumulates, over finished
 * episodes: count, sum episode_reward, sum episode_length, sum start loss,
 * sum final loss (the per-GPU input of the NCCL stats all-reduce). */
int lg_step(lg_env *env, const int64_t *actions_dev, void *obs_dev, double *reward_dev,
            uint8_t *done_dev, const lg_info *info, double *stats_dev, void *stream);
/* lg_step with flags: LG_STEP_NO_AUTO_RESET leaves finished envs as they are
 * (the scalar facade's _Core.step(auto_reset=False), env.py:611-630). */
#define LG_STEP_NO_AUTO_RESET 1u
/* LG_STEP_VALIDATE: check every action id on device first; if one is out of
 * range, LG_FLAG_BAD_ACTION is raised and the step kernel returns without
 * touching any env (the reference validates before mutating, env.py:358-361).
 * Read the verdict with lg_errors (one 4-byte read, the call's only sync). */
#define LG_STEP_VALIDATE 2u
int lg_step_flags(lg_env *env, const int64_t *actions_dev, void *obs_dev, double *reward_dev,
                  uint8_t *done_dev, const lg_info *info, double *stats_dev, uint32_t flags, void *stream);
/* BatchEnv.observe (env.py:587-588). */
int lg_observe(lg_env *env, void *obs_dev, void *stream);
/* The same step with HOST buffers: H2D of actions and D2H of every output
 * happen inside the call, which returns after the stream synchronises.
 * Observations without control planes cross PCIe packed (the kernel writes
 * the 0/1 planes as one bit stream, element t = bit t) in chunks, and the
 * library's host threads expand each chunk into obs_host (float32 or uint8,
 * any alignment, pinned or pageable) as soon as its copy lands: 1/32 of the
 * PCIe bytes of a float32 copy. LG_HOST_EXPAND=0 selects the plain copy. */
int lg_step_host(lg_env *env, const int64_t *actions_host, void *obs_host, double *reward_host,
                 uint8_t *done_host, const lg_info *info_host, void *stream);
/* Host threads lg_step_host expands observations with (LG_HOST_THREADS). */
int lg_host_threads(void);
/* Host-side expansion of a packed observation stream (LG_OBS_BITS layout,
 * element t = bit t%32 of word t/32) into n_elems float32 (fmt 0) or uint8
 * (fmt 1) 0/1 values at dst (any alignment). What lg_step_host does after the
 * copy; no GPU involved. */
int lg_unpack_host(const uint32_t *bits, int64_t n_elems, void *dst, int fmt);

/* Designer edits on imported states: recompute metrics + loss of the masked
 * envs (mask NULL = all) after their tiles/frozen planes changed (with_pin /
 * without_pin, env.py:657-667,684-715), or with reprice_only=1 only the loss
 * after a target change (with_target, env.py:670-681). */
int lg_recompute(lg_env *env, const uint8_t *mask_dev, int reprice_only, void *stream);

/* BatchEnv.state_dict / load_state_dict (env.py:535-585), device buffers. */
int lg_export_state(lg_env *env, const lg_state *dst_dev, void *stream);
int lg_import_state(lg_env *env, const lg_state *src_dev, void *stream);

/* Read and clear the device error flags (synchronises the stream). */
int lg_errors(lg_env *env, uint32_t *flags, void *stream);

/* harness.uniform_policy stand-in (harness.py:83-87): device-side uniform
 * actions in [0, n_actions) from a counter hash of (seed, global env index). */
int lg_random_actions(lg_env *env, int64_t *actions_dev, uint64_t seed, void *stream);

/* The random-policy loop of harness.bench_random_fps (harness.py:149-175:
 * rng.integers + BatchEnv.step) as one call: each env's action is the one
 * lg_random_actions(seed) would draw, recorded in actions_out when non-null,
 * then the env steps as lg_step. Consecutive lg_step_random calls of one env
 * on one stream, with no other call on that env between them, are chained:
 * each launch is a programmatic dependent launch of the previous one, and
 * its blocks wait per block (same envs, same block) instead of for the whole
 * previous grid, so the last wave of step k overlaps the start of step k+1.
 * Results are identical to lg_random_actions + lg_step. Other work the caller
 * enqueues on the stream between two chained calls must not write the env's
 * outputs (obs/reward/done/info/actions_out buffers). LG_NO_CHAIN=1 disables
 * the overlap. Maps wider or taller than 32 (64-row lane teams) draw the
 * actions with their own kernel and are not chained. */
int lg_step_random(lg_env *env, uint64_t seed, int64_t *actions_out_dev, void *obs_dev, double *reward_dev,
                   uint8_t *done_dev, const lg_info *info, double *stats_dev, void *stream);

/* harness.first_episode_rewards (harness.py:48-61), the per-step update on
 * device buffers of n envs: where done[b] && !seen[b], rewards[b] =
 * episode_reward[b] (the step's info["episode_reward"]) and seen[b] = 1;
 * n_seen (u64, device) counts the envs seen so far, so the caller polls one
 * word every few steps instead of the masks. Stream-ordered. */
int lg_first_episode(int64_t n, const uint8_t *done_dev, const double *episode_reward_dev, uint8_t *seen_dev,
                     double *rewards_dev, uint64_t *n_seen_dev, void *stream);

/* compute_metrics_batch (problems.py:105-129) on [B][H][W] stacks of tiles and
 * active masks; rng_dev [B][6] (advanced in place, binary only; may be NULL for
 * maze/dungeon); values_dev int64 [M][B], unreach_dev u8 [M][B]. */
int lg_metrics(int domain, int max_h, int max_w, int64_t n, const uint8_t *tiles_dev,
               const uint8_t *active_dev, uint64_t *rng_dev, int64_t *values_dev,
               uint8_t *unreach_dev, void *stream);

/* Policy consumer: the first layer of the reference's
 * ConvPolicy trunk (nets.py:150-183: Conv2d(C, K, 3) valid + ReLU) computed
 * straight from packed observation bits (LG_OBS_BITS layout, n_envs envs of
 * C x OH x OW elements). weight f32 [K][C][3][3], bias f32 [K] (device);
 * out [n_envs][K][OH-2][OW-2] (nhwc = 0) or [n_envs][OH-2][OW-2][K] (nhwc = 1,
 * the channels-last layout), float32 (out_bf16 = 0) or bfloat16 (1); nhwc = 2
 * is the tensor-core tile layout lg_policy_trunk reads (K = 16, bfloat16).
 * 1 <= K <= 64, C <= 16. Stream-ordered. */
int lg_conv1_bits(const uint32_t *bits_dev, int64_t n_envs, int C, int OH, int OW, const float *weight_dev,
                  const float *bias_dev, int K, void *out_dev, int out_bf16, int relu, int nhwc, void *stream);

/* Policy consumer, the rest of the default ConvPolicy trunk (nets.py:150-183,
 * conv_channels (16, 32), fc_dims (64,)) on the tensor cores (tcgen05, TMEM):
 * conv2 (16 -> 32, 3x3 valid) + ReLU, the 64-wide FC + ReLU and both heads,
 * for n_envs envs whose relu(conv1) is c1_tiles -- lg_conv1_bits with
 * nhwc = 2 (tile layout: [ceil(n/128)][P1*P1][128 envs x 16 ch] bf16 UMMA
 * core matrices), P1 = obs side - 2. w2 [9][512] and w3 [(P1-2)^2][2048]
 * are the conv2 / FC weights in the same bf16 layout (the Python mirror packs
 * them), b2 [32], b3 [64] f32; wh [n_actions + 1][64], bh [n_actions + 1] f32
 * = policy-head rows then the value head. Writes logits f32 [n][n_actions]
 * and value f32 [n]. n_actions <= 16. Stream-ordered. */
int lg_policy_trunk(const void *c1_tiles, int64_t n_envs, int P1, const void *w2, const float *b2, const void *w3,
                    const float *b3, const float *wh, const float *bh, int n_actions, float *logits, float *value,
                    void *stream);
/* lg_policy_trunk + the action draw of ppo.collect_rollout (ppo.py:125-130:
 * Categorical(logits).sample() and log_prob) in the heads' epilogue:
 * actions int64 [n], logp f32 [n] = log softmax(logits)[action]; the uniform
 * of env i is a counter hash of (seed, i), so one seed per step. */
int lg_policy_trunk_sample(const void *c1_tiles, int64_t n_envs, int P1, const void *w2, const float *b2,
                           const void *w3, const float *b3, const float *wh, const float *bh, int n_actions,
                           float *logits, float *value, uint64_t seed, int64_t *actions, float *logp, void *stream);

/* Host SeedSequence(seed).spawn(offset+n)[offset+i] -> rng [n][6] (env.py:591-594). */
int lg_seed_streams(uint64_t seed, int64_t offset, int64_t n, uint64_t *rng_host);

#ifdef __cplusplus
}
#endif
#endif
