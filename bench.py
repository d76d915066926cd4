"""Throughput bench of the batched PCGRL env step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1..c5] [--envs B]

A "step" is one pass of the hot path over the whole batch: device-side
uniform random actions (harness.uniform_policy, harness.py:83-87) + BatchEnv.step
(action apply, metric recompute, reward, auto-reset, observation write), as
timed by the reference harness (harness.py:149-175).

Default workload = config c5 (BASELINE.json configs[4]): binary 16x16 narrow,
obs 31x31, 2^20 environments in total, sharded over the N GPUs (strong
scaling: the global batch is fixed). The per-step observation output alone is
16.1 GB, far larger than L2 (126 MB), so no L2 flush is needed between steps.

For N > 1 run under torchrun (one process per GPU, NCCL); the timed region is
bracketed by a barrier + synchronize, and the max over ranks is reported.
``--impl reference`` times the CPU oracle port (oracle/, the reference's
algorithm restated in C, all host cores) on a bounded sample of the same
workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs -> EnvConfig kwargs and global env counts
CONFIGS = {
    "c1": ("binary 16x16 narrow, full-map obs 31, 64 envs", dict(domain="binary"), 64),
    "c2": ("maze 16x16 turtle, obs 31, 4096 envs", dict(domain="maze", representation="turtle"), 4096),
    "c3": ("dungeon 16x16 wide, pinpoints + randomized shapes, 65536 envs",
           dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
                randomize_shape=True), 65536),
    "c4": ("binary narrow obs 7x7 on 64x64 maps, 65536 envs",
           dict(domain="binary", max_width=64, max_height=64, obs_size=7), 65536),
    "c5": ("binary 16x16 narrow, obs 31, 2^20 envs sharded over the GPUs",
           dict(domain="binary"), 1 << 20),
}
METRIC = "env-steps/sec (binary 16x16 narrow) at 1/2/4/8 B200 vs host-CPU ref; HBM GB/s"
UNIT = "env-steps/s"


def algorithmic_bytes_per_env_step(obs_shape) -> int:
    """API-mandated I/O = obs write 4*C*OH*OW + action 8 (read
    by lg_step; drawn in-kernel and written out by lg_step_random) + reward
    write 8 + done write 1."""
    c, h, w = obs_shape
    return 4 * c * h * w + 8 + 8 + 1


def kernel_name(cfg, team: int) -> str:
    """The step kernel this config launches: the specialised instantiations
    (pcgrl_b200.cu spec_enabled / SoloKernel::spec) for the plain float32 path,
    else the generic one."""
    plain = (not cfg.controllable and not cfg.deterministic_metrics
             and os.environ.get("LG_NO_SPEC", "0")[:1] != "1")
    nopins = not cfg.pinpoints
    if team == 1:
        spec = plain and ((cfg.domain == "binary" and cfg.representation == "narrow" and nopins)
                          or (cfg.domain == "dungeon" and cfg.representation == "wide"))
        return f"env_solo_kernel_{cfg.domain}" + ("_s" if spec else "")
    if plain and nopins and cfg.domain == "binary" and cfg.representation == "narrow" \
            and max(cfg.max_width, cfg.max_height) > 32:
        return "env_kernel<G64, binary, spec narrow/no-pins>"
    if plain and nopins and team == 16 and cfg.domain == "maze" and cfg.representation == "turtle":
        return "env_kernel<G16, maze, spec turtle/no-pins>"
    return f"env_kernel<team {team}, {cfg.domain}>"


L2_BYTES = 126 * 2 ** 20
# st.global.cs.v8 stores only, 9472 blocks over 4 GB (profiles/r1_store_ceiling.txt)
STORE_CEILING_GBS = 7199.5


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_tensor_peak():
    """Dense bf16 TFLOP/s from MEASURED_PEAKS.json (cuBLAS), else the nominal 2250."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("bf16_tflops", "tensor_bf16_tflops", "bf16_dense_tflops"):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 2250.0


def load_traffic(config: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(config)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def rank_cpu_slice(local_rank: int, local_world: int, torch, dev):
    """The host cores this rank should use: its share of the cores of its
    GPU's NUMA node (ranks on the same node split them), else its share of
    the process's allowed cores. Returns a sorted list of cpu ids."""
    allowed = sorted(os.sched_getaffinity(0))
    if local_world <= 1:
        return allowed

    def node_of(i):
        try:
            pr = torch.cuda.get_device_properties(i)
            bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
                return int(f.read())
        except Exception:
            return -1

    def cpulist(node):
        cpus = set()
        try:
            with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
                for part in f.read().strip().split(","):
                    a, _, b = part.partition("-")
                    cpus.update(range(int(a), int(b or a) + 1))
        except Exception:
            return []
        return sorted(cpus & set(allowed))

    nodes = [node_of(i) for i in range(min(local_world, torch.cuda.device_count()))]
    mine = nodes[local_rank] if local_rank < len(nodes) else -1
    pool = cpulist(mine) if mine >= 0 else []
    peers = [i for i, n in enumerate(nodes) if n == mine] if pool else list(range(local_world))
    if not pool:
        pool = allowed
    k = max(1, len(pool) // max(1, len(peers)))
    j = peers.index(local_rank) if local_rank in peers else local_rank
    return pool[j * k:(j + 1) * k] or pool


def cpu_oracle_run(cfg, n_envs: int, steps: int, warmup: int, threads: int):
    """Time the CPU oracle (reference algorithm, C port) on the host cores."""
    import numpy as np
    from oracle import oracle as O

    O.set_threads(threads)
    env = O.OracleBatchEnv(cfg, n_envs, seed=0)
    env.reset()
    rng = np.random.default_rng(n_envs)
    obs = np.empty((n_envs,) + env.observation_shape, dtype=np.float32)
    for _ in range(warmup):
        env.step_no_obs(rng.integers(0, cfg.n_actions, size=n_envs))
        env.observe(obs)
    acts = [rng.integers(0, cfg.n_actions, size=n_envs) for _ in range(steps)]
    t0 = time.perf_counter()
    for a in acts:
        env.step_no_obs(a)
        env.observe(obs)
    dt = time.perf_counter() - t0
    return n_envs * steps / dt, dt


def run_reference(args, cfg, workload, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = args.cpu_envs or min(CONFIGS[args.config][2], 65536)
    value, dt = cpu_oracle_run(cfg, n, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8/int32/f64",
        "data": "synthetic (uniform random actions, seed 0)",
        "config": {"workload": workload, "config": args.config, "envs_sampled": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n} envs x {args.steps} steps of the same config "
                                   f"(oracle/ C restatement of levelgen BatchEnv.step+observe)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--envs", type=int, default=0, help="override the global env count")
    ap.add_argument("--cpu-envs", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-u8", action="store_true", help="skip the opt-in uint8-observation side run")
    ap.add_argument("--no-policy", action="store_true", help="skip the policy-rollout side run")
    ap.add_argument("--no-graph", action="store_true", help="time only the eager launch loop")
    ap.add_argument("--burn-in", type=int, default=-1,
                    help="untimed steps after warm-up (default: one full episode, 3*h*w)")
    ap.add_argument("--stats-every", type=int, default=10,
                    help="episode-stats all-reduce every S timed steps on a side stream (N > 1)")
    ap.add_argument("--no-proxy", action="store_true", help="skip the single-GPU scaling proxy")
    ap.add_argument("--policy-envs", type=int, default=65536)
    ap.add_argument("--policy-steps", type=int, default=8)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "RANK" in os.environ:
        # NCCL reads its debug settings once, when torch first touches it: set
        # them before torch is imported (communicator INIT lines: rank count)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world

    from paper_2408_12525_b200.config import EnvConfig
    desc, kw, default_b = CONFIGS[args.config]
    cfg = EnvConfig(**kw)
    global_b = args.envs or default_b
    workload = f"{args.config}: {desc}"

    if args.impl == "reference":
        run_reference(args, cfg, workload, rank)
        return

    import torch
    import torch.distributed as dist

    # LG_BENCH_SAME_DEVICE=1: every rank on cuda:0 -- a functional test of the
    # N > 1 code path on a one-GPU box (tests/test_gpu_bench_contract.py, gloo);
    # never a measurement
    dev_index = 0 if os.environ.get("LG_BENCH_SAME_DEVICE") == "1" else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    all_cpus = sorted(os.sched_getaffinity(0))
    cpus = rank_cpu_slice(local_rank, local_world, torch, dev)
    if local_world > 1:
        # each rank expands its own observations on its own cores (no
        # oversubscription: 8 ranks x all cores would thrash the host)
        try:
            os.sched_setaffinity(0, cpus)
        except Exception:
            pass
        os.environ.setdefault("LG_HOST_THREADS", str(len(cpus)))
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ or "MASTER_ADDR" in os.environ
    if distributed:
        # communicator setup is logged so the rank count can be checked. NCCL
        # (and torch's NCCL banner) write to file descriptor 1: point it at
        # stderr for the whole run and keep Python's stdout on the original
        # descriptor, so stdout carries only the one JSON line.
        sys.stdout.flush()
        out_fd = os.dup(1)
        os.dup2(2, 1)
        sys.stdout = os.fdopen(out_fd, "w", buffering=1)
        backend = os.environ.get("LG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        print(f"[bench] rank {rank}/{world}: {backend} communicator of {dist.get_world_size()} ranks on {dev}",
              file=sys.stderr, flush=True)
    from paper_2408_12525_b200 import _lib
    from paper_2408_12525_b200.env import INFO_KEYS, BatchEnv, NumpyBatchEnv

    from paper_2408_12525_b200.sharding import STAT_NAMES, EpisodeStats, max_over_ranks, shard
    offset, B = shard(global_b, world, rank)
    env = BatchEnv(cfg, B, seed=0, device=dev, global_offset=offset, validate=False)
    # Output slots: a step's outputs (obs, actions, reward, done, info) smaller
    # than L2 would be rewritten in place in L2 step after step and never
    # reach HBM. Those configs rotate R output slots, R x the step's output
    # >= 3x L2 (capped at K), as a rollout buffer does ([T, B] in
    # ppo.collect_rollout), so consecutive steps write cold lines.
    c_, h_, w_ = env.observation_shape
    out_bytes = B * (4 * c_ * h_ * w_ + 8 + 8 + 1 + 1 + 8 + 8 + 8 + 8)
    n_slots = 1 if out_bytes >= 2 * L2_BYTES else max(1, min(args.steps, -(-3 * L2_BYTES // out_bytes)))
    slots = [dict(obs=env.new_obs(), acts=torch.empty(B, dtype=torch.int64, device=dev),
                  reward=torch.empty(B, dtype=torch.float64, device=dev),
                  done=torch.empty(B, dtype=torch.bool, device=dev), info=env._info_buffers())
             for _ in range(n_slots)]
    obs, acts, reward, done, info = (slots[0][k] for k in ("obs", "acts", "reward", "done", "info"))
    ep_stats = EpisodeStats(dev)
    stats = ep_stats.t
    env.reset(out=obs)
    stream = torch.cuda.current_stream(dev)

    # One step of harness.bench_random_fps's loop (harness.py:149-175): a
    # uniform action per env, then the batched step. lg_step_random draws the
    # actions in the step kernel (recorded in `acts`, the same values
    # lg_random_actions writes) and chains consecutive launches: step k+1's
    # blocks start while step k's last wave runs (include/pcgrl_b200.h).
    def one_step(i):
        o = slots[i % n_slots]
        env.step_random(1_000_003 * i + 17, o["obs"], o["reward"], o["done"], o["info"], stats,
                        actions_out=o["acts"])

    for i in range(args.warmup):
        one_step(i)
    # Burn-in (untimed): run one full episode past warm-up, so the timed
    # window is steady state with every env's first auto-reset behind it.
    # Lockstep configs (fixed shape, no change budget: c1/c2/c4/c5) reset all
    # envs on the same step, L = 3*h*w; that step's cost is timed here and
    # reported as episode_boundary.
    H, W = cfg.max_height, cfg.max_width
    ep_len = int(cfg.max_steps or 3 * H * W)
    burn = args.burn_in if args.burn_in >= 0 else ep_len
    lockstep = not cfg.randomize_shape and not cfg.change_budget
    bev = []
    for i in range(burn):
        j = args.warmup + i
        if lockstep:
            bev.append((j + 1, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            bev[-1][1].record(stream)
        one_step(j)
        if lockstep:
            bev[-1][2].record(stream)
    torch.cuda.synchronize()
    boundary = None
    if lockstep and bev:
        times = {k: a.elapsed_time(b) for k, a, b in bev}
        if ep_len in times:
            steady = statistics.median(v for k, v in times.items() if k % ep_len)
            t_reset = times[ep_len]
            boundary = {"step": ep_len, "reset_step_ms": t_reset, "steady_step_ms_events": steady,
                        "note": "every env of the lockstep batch auto-resets on step 3*h*w; both timed with "
                                "per-step events during the burn-in (which break the launch chain); "
                                "amortized = one episode cycle of L-1 steps at the timed rate + the reset step"}
    t0_step = args.warmup + burn
    if world > 1:
        dist.barrier()
    clk = ClockSampler(dev_index)
    clk.start()
    time.sleep(0.3)
    K = args.steps
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # N > 1: the episode counters are all-reduced every S steps on a side
    # stream (NCCL over NVLink), off the step's critical path
    side = torch.cuda.Stream(dev) if world > 1 else None
    snap = torch.zeros_like(stats)
    red_ev = []
    t_start.record(stream)
    for i in range(K):
        one_step(i + t0_step)
        if side is not None and (i + 1) % args.stats_every == 0:
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                snap.copy_(stats)
                r0.record(side)
                dist.all_reduce(snap)
                r1.record(side)
                red_ev.append((r0, r1))
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reduce_info = None
    if red_ev:
        rms = [a.elapsed_time(b) for a, b in red_ev]
        reduce_info = {"every_steps": args.stats_every, "count": len(rms), "mean_ms": sum(rms) / len(rms),
                       "max_ms": max(rms), "stream": "side (overlaps the step kernels)",
                       "global_episodes_seen": float(snap[0])}
    elapsed_ms = t_start.elapsed_time(t_end)
    elapsed_ms = max_over_ranks(elapsed_ms, dev)
    step_ms = elapsed_ms / K  # one step kernel per step
    eager_ms = elapsed_ms
    graph_ms = None
    eager_step_ms = kernel_graph_ms = None
    split = None
    if not args.no_graph:
        # the same K steps (fresh seeds) captured once in a CUDA graph and
        # replayed: no per-launch CPU gaps, which matter for the small configs
        # (c1: 64 envs, ~20 us kernels). The graph holds exactly the K chained
        # step launches, so its span / K is also the step kernel's time.
        g = torch.cuda.CUDAGraph()
        base = t0_step + K
        with torch.cuda.graph(g):
            for i in range(K):
                one_step(base + i)
        g.replay()  # warm replay (K more steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        graph_ms = max_over_ranks(g0.elapsed_time(g1), dev)
        if world == 1:  # N > 1: the eager loop carries the stats all-reduce; it is the value
            elapsed_ms = min(elapsed_ms, graph_ms)
        del g
        kernel_graph_ms = graph_ms / K
        eager_step_ms = step_ms
        step_ms = min(step_ms, kernel_graph_ms)
        # For contrast: the unfused loop -- lg_random_actions, then lg_step on
        # those actions (two launches per step, each waiting for the whole
        # previous grid), same graph timing.
        gs = torch.cuda.CUDAGraph()
        base = t0_step + 3 * K
        with torch.cuda.graph(gs):
            for i in range(K):
                o = slots[(base + i) % n_slots]
                env.random_actions(1_000_003 * (base + i) + 17, out=o["acts"])
                env.step_raw(o["acts"], o["obs"], o["reward"], o["done"], o["info"], stats)
        gs.replay()
        torch.cuda.synchronize()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        gs.replay()
        k1.record(stream)
        torch.cuda.synchronize()
        split_ms = max_over_ranks(k0.elapsed_time(k1), dev) / K
        del gs
        split = {"value": global_b / (split_ms / 1e3), "ms_per_step": split_ms,
                 "launches_per_step": 2,
                 "note": "lg_random_actions + lg_step per step (no launch chaining), CUDA-graph replay"}
    clocks = clk.stop()
    ep_stats.all_reduce()  # the episode-stats reduce (NCCL over NVLink when N > 1)
    stats_host = [float(x) for x in stats.cpu()]
    errs = env.errors()
    if errs:
        raise SystemExit(f"device error flags {errs}")
    value = global_b * K / (elapsed_ms / 1e3)
    if boundary:
        L, steady_ms = boundary["step"], elapsed_ms / K
        boundary["amortized_value"] = global_b * L / (((L - 1) * steady_ms + boundary["reset_step_ms"]) / 1e3)

    obs_shape = env.observation_shape
    team = env._desc.team
    bytes_step = algorithmic_bytes_per_env_step(obs_shape)
    peak, peak_kind = load_peaks()
    achieved_gbs = B * bytes_step / (step_ms / 1e3) / 1e9

    # end to end through the public numpy API: H2D actions from pinned host
    # memory, D2H of obs/reward/done/info into host arrays, every step. The
    # observations cross PCIe as packed 0/1 bit planes (1 bit per element) and
    # the library's host threads expand them into the caller's float32 array
    # (lg_step_host); LG_HOST_EXPAND=0 gives the plain float32 copy for contrast.
    import numpy as np

    def e2e_run(obs_dtype: str, packed: bool, fresh: bool = False):
        if packed:
            os.environ.pop("LG_HOST_EXPAND", None)  # the library's default choice
        else:
            os.environ["LG_HOST_EXPAND"] = "0"
        torch.cuda.empty_cache()
        # fresh=False: pinned output arrays reused across steps (the caller
        # copies what it keeps, as ppo.collect_rollout does, ppo.py:131);
        # fresh=True: new pageable numpy arrays every step, the reference's
        # ownership contract (env.py:233)
        nenv = NumpyBatchEnv(cfg, B, seed=0, device=dev, global_offset=offset, pinned=not fresh, copy=fresh,
                             obs_dtype=obs_dtype)
        nenv.reset()
        rng = np.random.default_rng(1)
        a0 = rng.integers(0, cfg.n_actions, size=B)
        nenv.step(a0)  # warm-up (allocations)
        t0 = time.perf_counter()
        nenv.step(a0)  # sizes the timed loop
        per = time.perf_counter() - t0
        # at least e2e_steps steps and ~1.5 s of them (host-memory-bound: one
        # short sample is noisy; small batches are microseconds per step)
        n_steps = max(args.e2e_steps, min(2000, int(1.5 / max(per, 1e-6))))
        if fresh and per > 0.5:
            n_steps = 3
        if world > 1:
            n_steps = int(max_over_ranks(float(n_steps), dev))
        host_acts = [rng.integers(0, cfg.n_actions, size=B) for _ in range(n_steps)]
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = None
        for a in host_acts:
            res = nenv.step(a)  # a caller holds a step's arrays until the next step returns
        dt = max_over_ranks(time.perf_counter() - t0, dev)
        del res
        del nenv
        os.environ.pop("LG_HOST_EXPAND", None)
        n_el = B * int(np.prod(env.observation_shape))
        # the library packs when there are no control planes and the float32
        # observation is >= 2 MB (below that the plain copy has lower latency)
        # (below that only into pageable arrays: the fresh-array run)
        use_packed = packed and not cfg.controllable and (n_el * 4 >= (2 << 20) or fresh)
        obs_d2h = (n_el + 31) // 32 * 4 if use_packed else n_el * (1 if obs_dtype == "uint8" else 4)
        d2h = obs_d2h + B * (8 + 1 + 1 + 8 + 8 + 8 + 8)
        out = {"value": global_b * n_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": B * 8, "d2h_bytes_per_step": d2h, "steps": n_steps,
               "pcie_d2h_gbs": d2h * n_steps / dt / 1e9,
               "api": "NumpyBatchEnv.step -> lg_step_host " +
                      ("(fresh pageable arrays every step, copy=True)" if fresh else
                       "(pinned arrays reused across steps, copy=False)")}
        if use_packed:
            out["transfer"] = (f"packed 0/1 bit planes D2H, expanded to {obs_dtype} in the caller's array "
                               f"by {_lib.load().lg_host_threads()} host threads (non-temporal stores)")
        else:
            out["transfer"] = f"{obs_dtype} observation copy D2H"
        return out

    def e2e_device_obs():
        # A GPU-side consumer's loop (a policy on the same device): numpy
        # actions from pinned host memory in, observations left on the device,
        # reward and done read back to the host every step. Side figure: the
        # reference's contract returns the observation in host memory (e2e above).
        torch.cuda.empty_cache()
        denv = BatchEnv(cfg, B, seed=0, device=dev, global_offset=offset, validate=False)
        dobs = denv.new_obs()
        denv.reset(out=dobs)
        rng = np.random.default_rng(2)
        n_steps = 20
        host_acts = [torch.from_numpy(rng.integers(0, cfg.n_actions, size=B)).pin_memory() for _ in range(n_steps + 1)]
        d_act = torch.empty(B, dtype=torch.int64, device=dev)
        d_rew = torch.empty(B, dtype=torch.float64, device=dev)
        d_done = torch.empty(B, dtype=torch.bool, device=dev)
        h_rew = torch.empty(B, dtype=torch.float64).pin_memory()
        h_done = torch.empty(B, dtype=torch.bool).pin_memory()

        def one(a):
            d_act.copy_(a, non_blocking=True)
            denv.step_raw(d_act, dobs, d_rew, d_done)
            h_rew.copy_(d_rew, non_blocking=True)
            h_done.copy_(d_done, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

        one(host_acts[-1])
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for a in host_acts[:n_steps]:
            one(a)
        dt = max_over_ranks(time.perf_counter() - t0, dev)
        del denv, dobs
        return {"value": global_b * n_steps / dt, "unit": UNIT, "h2d_bytes_per_step": B * 8,
                "d2h_bytes_per_step": B * 9, "steps": n_steps,
                "api": "BatchEnv.step_raw with pinned host actions; observation stays on the device; "
                       "reward + done D2H and a host sync every step",
                "note": "side figure for GPU-resident consumers, not the reference's host-array contract"}

    e2e = None
    if not args.no_e2e:
        del obs
        e2e = e2e_run("float32", True)
        e2e["float32_copy"] = e2e_run("float32", False)
        e2e["fresh_arrays"] = e2e_run("float32", True, fresh=True)
        e2e["device_obs"] = e2e_device_obs()

    # Side measurement (does not change the headline): the same workload with
    # the opt-in uint8 observation format (4x fewer bytes per env-step).
    u8 = None
    if not args.no_u8 and not cfg.controllable:
        import torch as _t
        _t.cuda.empty_cache()
        env8 = BatchEnv(cfg, B, seed=0, device=dev, global_offset=offset, validate=False, obs_dtype="uint8")
        out8 = B * (c_ * h_ * w_ + 17)  # the same rule as the float32 run: cold output lines
        n8 = 1 if out8 >= 2 * L2_BYTES else max(1, min(K, -(-3 * L2_BYTES // out8)))
        obs8s = [env8.new_obs() for _ in range(n8)]
        obs8 = obs8s[0]
        env8.reset(out=obs8)
        for i in range(args.warmup):
            env8.step_random(1_000_003 * i + 17, obs8, reward, done, info, None, actions_out=acts)
        torch.cuda.synchronize()
        e80, e81 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e80.record(stream)
        for i in range(K):
            o = slots[i % n_slots]
            env8.step_random(1_000_003 * (i + args.warmup) + 17, obs8s[i % n8], o["reward"], o["done"], o["info"],
                             None, actions_out=o["acts"])
        e81.record(stream)
        torch.cuda.synchronize()
        ms8 = max_over_ranks(e80.elapsed_time(e81) / K, dev)
        c_, h_, w_ = env8.observation_shape
        bytes8 = c_ * h_ * w_ + 17
        u8 = {"value": global_b / (ms8 / 1e3), "unit": UNIT, "step_kernel_ms": ms8,
              "bytes_per_env_step": bytes8, "achieved_gbs": B * bytes8 / (ms8 / 1e3) / 1e9,
              "frac_of_peak": B * bytes8 / (ms8 / 1e3) / 1e9 / peak,
              "note": "opt-in obs_dtype='uint8' (same 0/1 planes); not the reference float32 contract"}
        u8["output_slots"] = n8
        del obs8, obs8s, env8
        if not args.no_e2e:
            u8["e2e"] = e2e_run("uint8", True)

    # Side measurement (does not change the headline): the
    # policy consumer in the loop -- ppo.collect_rollout on device (ConvPolicy
    # forward, multinomial sampling, env step, rollout buffer) with (a) the
    # reference's float32 observations + torch conv trunk, (b) the same with
    # bf16 autocast, (c) packed observation bits + lg_conv1_bits first layer +
    # bf16 rest. Fewer envs than the headline (the conv trunk dominates).
    pol = None
    if not args.no_policy and not cfg.controllable and cfg.representation != "wide":
        from paper_2408_12525_b200.policy import PackedPolicy, collect_rollout, default_arch, init_policy
        torch.cuda.empty_cache()
        Bp = min(B, args.policy_envs)
        pol = {"envs": Bp, "steps": args.policy_steps, "unit": UNIT,
               "note": "ppo.collect_rollout on device: policy forward + sampling + env step + rollout buffer"}

        def rollout_rate(fmt, make_policy):
            e = BatchEnv(cfg, Bp, seed=0, device=dev, global_offset=offset, validate=False, obs_dtype=fmt)
            o = e.reset()
            shp = e.observation_shape
            model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).to(dev)
            p_ = make_policy(model, shp)
            gen = torch.Generator(device=dev).manual_seed(0)
            _, o, _ = collect_rollout(p_, e, 2, gen, o)  # warm-up (cuDNN autotune, allocations)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            collect_rollout(p_, e, args.policy_steps, gen, o)
            a1.record()
            torch.cuda.synchronize()
            ms = a0.elapsed_time(a1)
            del e, model, p_
            torch.cuda.empty_cache()
            return Bp * args.policy_steps / (ms / 1e3)

        def autocast_policy(model, shp):
            def f(x):
                with torch.autocast("cuda", dtype=torch.bfloat16):
                    lg, v = model(x)
                return lg.float(), v.float()
            return f

        # the first conv alone: lg_conv1_bits from packed bits vs cuDNN on float32 obs
        from paper_2408_12525_b200.policy import conv1_bits
        e = BatchEnv(cfg, Bp, seed=0, device=dev, global_offset=offset, validate=False, obs_dtype="bits")
        bits_o = e.reset()
        shp = e.observation_shape
        m0 = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).to(dev)
        conv = m0.trunk[0]
        from paper_2408_12525_b200.env import unpack_obs
        obs_f = unpack_obs(bits_o, Bp, shp)

        def time_ms(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(reps):
                fn()
            a1.record()
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps

        K_, P_ = conv.weight.shape[0], (shp[1] - 2) * (shp[2] - 2)
        n_in = Bp * shp[0] * shp[1] * shp[2]
        with torch.no_grad():
            t_f32 = time_ms(lambda: conv1_bits(bits_o, Bp, shp, conv.weight, conv.bias))
            t_bf = time_ms(lambda: conv1_bits(bits_o, Bp, shp, conv.weight, conv.bias, out_dtype=torch.bfloat16))
            t_cud = time_ms(lambda: torch.relu(conv(obs_f)))
        by_f32 = Bp * K_ * P_ * 4 + n_in / 8
        by_bf = Bp * K_ * P_ * 2 + n_in / 8
        pol["conv1"] = {
            "lg_conv1_bits_f32_ms": t_f32, "lg_conv1_bits_f32_gbs": by_f32 / t_f32 / 1e6,
            "lg_conv1_bits_bf16_ms": t_bf, "lg_conv1_bits_bf16_gbs": by_bf / t_bf / 1e6,
            "cudnn_f32_obs_ms": t_cud, "frac_of_peak_bf16": by_bf / t_bf / 1e6 / peak,
            "note": "bytes = output + packed input (1 bit/element); cuDNN reads float32 obs"}
        del e, m0, conv, obs_f, bits_o
        torch.cuda.empty_cache()

        # the default trunk on the tensor cores: lg_conv1_bits (bf16 tiles) +
        # lg_policy_trunk (conv2 + FC as tcgen05 MMAs with TMEM accumulators, heads)
        from paper_2408_12525_b200.policy import TrunkPolicy
        e = BatchEnv(cfg, Bp, seed=0, device=dev, global_offset=offset, validate=False, obs_dtype="bits")
        bits_o = e.reset()
        shp = e.observation_shape
        m0 = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).to(dev)
        tp = TrunkPolicy(m0, shp)
        c1t = tp.conv1_tiles(bits_o, Bp)
        t_c1t = time_ms(lambda: tp.conv1_tiles(bits_o, Bp))
        t_tp = time_ms(lambda: tp(bits_o, Bp)) - t_c1t
        P2 = shp[1] - 4
        tflop = Bp * (P2 * P2 * 32 * 16 * 9 * 2 + 32 * P2 * P2 * 64 * 2) / 1e12
        tf_peak = load_tensor_peak()
        pol["tcgen05_trunk"] = {
            "conv1_tiles_ms": t_c1t, "conv1_tiles_gbs": c1t.numel() * 2 / t_c1t / 1e6,
            "trunk_ms": t_tp, "trunk_tflops": tflop / (t_tp / 1e3), "tensor_peak_tflops": tf_peak,
            "frac_of_tensor_peak": tflop / (t_tp / 1e3) / tf_peak if tf_peak else None,
            "note": "conv2 (16->32, 3x3) + FC (32*P2^2 -> 64) algorithmic flops; bf16 operands, fp32 accumulate"}
        del e, m0, tp, c1t, bits_o
        torch.cuda.empty_cache()
        pol["bits_obs_tcgen05_trunk"] = rollout_rate("bits", lambda m, shp: TrunkPolicy(m, shp))
        pol["float32_obs_torch_f32"] = rollout_rate("float32", lambda m, shp: m)
        pol["float32_obs_torch_bf16"] = rollout_rate("float32", autocast_policy)
        pol["bits_obs_conv1_bits_bf16"] = rollout_rate("bits", lambda m, shp: PackedPolicy(m, shp, bf16=True))
        pol["bits_obs_conv1_bits_bf16_nhwc"] = rollout_rate(
            "bits", lambda m, shp: PackedPolicy(m, shp, bf16=True, channels_last=True))

    # Single-GPU proxy of the strong-scaling sweep (c5): the per-GPU shard of
    # 2^20 envs at N = 2, 4, 8 run alone on this GPU (graph replay of K steps).
    proxy = None
    if world == 1 and not args.no_proxy and args.config == "c5":
        del env
        torch.cuda.empty_cache()
        proxy = {"note": "per-GPU rate of the N-GPU shard, measured on one B200; "
                         "projected speed-up = N * rate(shard) / value"}
        for n_gpu in (2, 4, 8):
            Bs = global_b // n_gpu
            pe = BatchEnv(cfg, Bs, seed=0, device=dev, validate=False)
            po = pe.new_obs()
            pa = torch.empty(Bs, dtype=torch.int64, device=dev)
            pr = torch.empty(Bs, dtype=torch.float64, device=dev)
            pd = torch.empty(Bs, dtype=torch.bool, device=dev)
            pe.reset(out=po)
            for i in range(args.warmup):
                pe.step_random(i, po, pr, pd, actions_out=pa)
            gp = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gp):
                for i in range(K):
                    pe.step_random(100 + i, po, pr, pd, actions_out=pa)
            gp.replay()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            gp.replay()
            g1.record(stream)
            torch.cuda.synchronize()
            rate = Bs * K / (g0.elapsed_time(g1) / 1e3)
            proxy[f"n{n_gpu}"] = {"envs_per_gpu": Bs, "per_gpu_value": rate,
                                  "projected_speedup": n_gpu * rate / value}
            del gp, pe, po, pa, pr, pd
            torch.cuda.empty_cache()

    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the oracle on all of the host's cores (rank 0, after the GPU work)
        try:
            os.sched_setaffinity(0, all_cpus)
        except Exception:
            pass
        threads = len(all_cpus)
        n_cpu = args.cpu_envs or min(global_b, 65536)
        # size the sample to roughly cpu-seconds of work
        v0, dt0 = cpu_oracle_run(cfg, n_cpu, 2, 1, threads)
        steps_cpu = max(2, int(args.cpu_seconds / max(dt0 / 2, 1e-3)))
        steps_cpu = min(steps_cpu, 200)
        v, dt = cpu_oracle_run(cfg, n_cpu, steps_cpu, 1, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n_cpu} envs x {steps_cpu} steps ({dt:.1f} s) of {args.config}; "
                         f"oracle/ C restatement of levelgen BatchEnv.step+observe, OpenMP"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8/int32/f64 (obs f32)",
            "data": "synthetic (device uniform random actions; env streams SeedSequence(0).spawn)",
            "config": {"workload": workload, "config": args.config, "global_envs": global_b,
                       "envs_per_gpu": B, "obs_shape": list(obs_shape),
                       "parallelism": f"env-sharded x{world}", "burn_in_steps": burn,
                       "l2": ("no flush: per-step output (%.3f GB) >> 126 MB L2" % (out_bytes / 1e9))
                       if n_slots == 1 else
                       ("no flush: per-step output %.1f MB < L2, rotated over %d output slots "
                        "(%.0f MB per cycle)" % (out_bytes / 1e6, n_slots, n_slots * out_bytes / 1e6)),
                       "output_slots": n_slots},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                         "frac": achieved_gbs / peak, "traffic": load_traffic(args.config),
                         "peak_kind": peak_kind, "frac_of_8000_nominal": achieved_gbs / 8000.0,
                         # the step's bytes are >99.9% writes: the copy peak (read+write) is
                         # not its ceiling; the measured streaming-store ceiling is
                         "store_ceiling_gbs": STORE_CEILING_GBS,
                         "frac_of_store_ceiling": achieved_gbs / STORE_CEILING_GBS,
                         "kernel": kernel_name(cfg, team) + " (fused step + obs)",
                         "bytes_per_env_step": bytes_step, "step_kernel_ms": step_ms,
                         "step_kernel_ms_from": "CUDA-graph replay of K chained step launches (events around "
                                                "it) / K: consecutive launches overlap at block granularity"
                         if kernel_graph_ms is not None and step_ms == kernel_graph_ms else "eager launch loop / K",
                         "step_kernel_ms_eager": eager_step_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # lg_step_random: one step kernel per step; maps over 32 rows/columns
            # (64-row lane teams, not chained) also launch random_actions_kernel
            "gpu_launches": K * (2 if max(cfg.max_width, cfg.max_height) > 32 else 1),
            "unchained_split_launch": split,
            "timing": {"eager_ms_per_step": eager_ms / K,
                       "graph_ms_per_step": graph_ms / K if graph_ms is not None else None,
                       "value_from": "graph" if graph_ms is not None and graph_ms <= eager_ms else "eager",
                       "note": "value = K steps / min(eager launch loop, one CUDA-graph replay of K "
                               "steps); both time the same work on the device"},
            "obs_uint8": u8,
            "policy_rollout": pol,
            "clocks": clocks,
            "episode_stats": dict(zip(STAT_NAMES, stats_host)),
            "episode_boundary": boundary,
            "stats_all_reduce": reduce_info,
            "scaling_proxy": proxy,
            "host": {"cpus_used_by_rank0": len(cpus), "local_world": local_world,
                     "comm": f"{os.environ.get('LG_BENCH_BACKEND', 'nccl')} x{world}" if distributed else "none"},
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
