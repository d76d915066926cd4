"""Episode runners, the evaluation grid and the random baseline on the GPU.

Mirror of ``levelgen.harness`` (reference harness.py) for the callers of the
env step that evaluate rather than train:

* ``first_episode_rewards`` (harness.py:48-61): steps a ``BatchEnv`` until
  every env has finished one episode and returns each env's first episode
  reward. The per-step bookkeeping runs on device (``lg_first_episode``: one
  kernel updates the seen mask, the rewards and a counter), so the host polls
  one 8-byte word every ``check_every`` steps instead of syncing on masks.
* ``greedy_policy`` / ``sampling_policy`` / ``uniform_policy``
  (harness.py:64-87): action functions. The policy ones run the ConvPolicy on
  the env's device (TF32 off, float32 as the reference); ``uniform_policy``
  draws from the caller's numpy Generator exactly as the reference does, so
  random-action runs are bit-identical to it.
* ``evaluate`` (harness.py:275-342) with ``EvalCell`` / ``EvalReport`` and
  their JSON/CSV encodings (harness.py:194-272), ``random_baseline``
  (harness.py:376-386), ``bench_random_fps`` (harness.py:149-175, device
  random actions).

Envs built here are stepped with ``validate=False`` (no per-step sync); their
error flags are read at every poll and raised as the reference would
(``ValueError`` from reset_rows).
"""
from __future__ import annotations

import contextlib
import csv
import io
import json
import os
import platform
import time
from dataclasses import asdict, dataclass, replace
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .config import EnvConfig
from .env import BatchEnv, _ptr, _stream

BENCH_LADDER = (1, 10, 50, 100, 200, 400, 600)
EVAL_WIDTHS = (8, 16, 24, 32)

ActFn = Callable[[object], object]


def _torch():
    import torch
    return torch


def machine_descriptor() -> dict[str, str]:
    """harness.machine_descriptor (harness.py:35-42), plus the GPU."""
    torch = _torch()
    d = {"platform": platform.platform(), "python": platform.python_version(), "numpy": np.__version__,
         "torch": torch.__version__, "cpus": str(os.cpu_count() or 1)}
    if torch.cuda.is_available():
        d["gpu"] = torch.cuda.get_device_name()
    return d


# ---------------------------------------------------------------------------
# episode runners
# ---------------------------------------------------------------------------


def first_episode_rewards(env: BatchEnv, act_fn: ActFn, *, check_every: int = 1) -> np.ndarray:
    """Step the batch until every env has finished one episode; return each
    env's first episode reward (float64 [n_envs], numpy) -- harness.py:48-61.

    ``act_fn(obs)`` gets the device observation tensor and returns actions
    (a device tensor or a numpy array). Envs that restart early keep stepping,
    so the batch stays lockstep-deterministic. With ``check_every == 1`` the
    env stops on exactly the reference's step; larger values poll less often
    and may step the (then discarded) batch a few steps further -- the
    returned rewards are the same.
    """
    torch = _torch()
    lib = _lib.load()
    B, dev = env.n_envs, env.device
    rewards = torch.zeros(B, dtype=torch.float64, device=dev)
    seen = torch.zeros(B, dtype=torch.uint8, device=dev)
    n_seen = torch.zeros(1, dtype=torch.int64, device=dev)
    obs = env.reset()
    check_every = max(1, int(check_every))
    while True:
        for _ in range(check_every):
            obs, _, done, info = env.step(act_fn(obs))
            with torch.cuda.device(dev):
                _lib.check(lib.lg_first_episode(B, _ptr(done), _ptr(info["episode_reward"]), _ptr(seen),
                                                _ptr(rewards), _ptr(n_seen), _stream(torch, dev)))
        if not env.validate:
            env.check_errors()
        if int(n_seen.item()) >= B:
            return rewards.cpu().numpy()


@contextlib.contextmanager
def _float32_exact():
    """The reference evaluates in float32 on the CPU: keep cuDNN/cuBLAS off TF32."""
    torch = _torch()
    old = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = old


def greedy_policy(model) -> ActFn:
    """harness.greedy_policy (harness.py:64-70): argmax of the logits."""
    torch = _torch()

    def act(obs):
        with torch.no_grad(), _float32_exact():
            logits, _ = model(obs)
        return logits.argmax(dim=-1)

    return act


def sampling_policy(model, sampler) -> ActFn:
    """harness.sampling_policy (harness.py:73-80): one multinomial draw per env
    from softmax(logits) with the caller's torch Generator (on the env's device)."""
    torch = _torch()

    def act(obs):
        with torch.no_grad(), _float32_exact():
            logits, _ = model(obs)
            probs = torch.softmax(logits, dim=-1)
        return torch.multinomial(probs, 1, generator=sampler).squeeze(1)

    return act


def uniform_policy(n_actions: int, rng: np.random.Generator) -> ActFn:
    """harness.uniform_policy (harness.py:83-87): the caller's numpy stream, as
    the reference draws it (the batch's actions cross PCIe, 8 bytes per env)."""
    def act(obs):
        return rng.integers(0, n_actions, size=obs.shape[0]).astype(np.int64)

    return act


# ---------------------------------------------------------------------------
# throughput (harness.py:90-175)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BenchRow:
    domain: str
    n_envs: int
    steps: int
    seconds: float
    fps: float


@dataclass
class BenchReport:
    machine: dict
    rows: list

    def fps_at(self, n_envs: int) -> float:
        for row in self.rows:
            if row.n_envs == n_envs:
                return row.fps
        raise KeyError(f"no ladder point at {n_envs} envs")

    def to_json(self) -> str:
        return json.dumps({"machine": self.machine, "rows": [asdict(r) for r in self.rows]}, indent=2)

    @classmethod
    def from_json(cls, text: str) -> "BenchReport":
        d = json.loads(text)
        return cls(machine=d["machine"], rows=[BenchRow(**r) for r in d["rows"]])


def bench_random_fps(domain: str, env_counts: Sequence[int] = BENCH_LADDER, seconds: float = 2.0, *,
                     config: EnvConfig | None = None, seed: int = 0, device=None) -> BenchReport:
    """harness.bench_random_fps (harness.py:149-175) on the GPU: uniform random
    actions generated on device (lg_random_actions), 3 warm-up steps, then
    steps for ``seconds`` of wall time; fps = env-steps / elapsed."""
    if not env_counts:
        raise ValueError("env_counts must be non-empty")
    torch = _torch()
    cfg = config or EnvConfig(domain=domain)
    rows = []
    for n in env_counts:
        env = BatchEnv(cfg, n, seed=seed, device=device, validate=False)
        obs = env.new_obs()
        acts = torch.empty(n, dtype=torch.int64, device=env.device)
        reward = torch.empty(n, dtype=torch.float64, device=env.device)
        done = torch.empty(n, dtype=torch.bool, device=env.device)
        env.reset(out=obs)
        k = 0
        for _ in range(3):
            env.random_actions(seed + k, out=acts)
            env.step_raw(acts, obs, reward, done)
            k += 1
        torch.cuda.synchronize(env.device)
        steps = 0
        t0 = time.perf_counter()
        while True:
            for _ in range(16):
                env.random_actions(seed + k, out=acts)
                env.step_raw(acts, obs, reward, done)
                k += 1
                steps += n
            torch.cuda.synchronize(env.device)
            elapsed = time.perf_counter() - t0
            if elapsed >= seconds:
                break
        env.check_errors()
        rows.append(BenchRow(domain=domain, n_envs=n, steps=steps, seconds=elapsed, fps=steps / elapsed))
    return BenchReport(machine=machine_descriptor(), rows=rows)


# ---------------------------------------------------------------------------
# evaluation grid (harness.py:182-342)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class EvalCell:
    obs_size: int
    trained_rand_shape: bool
    eval_rand_shape: bool
    width: int
    episodes: int
    mean: float
    std: float


@dataclass
class EvalReport:
    domain: str
    checkpoint_step: int
    n_seeds: int
    episodes_per_seed: int
    cells: list

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=2)

    @classmethod
    def from_json(cls, text: str) -> "EvalReport":
        d = json.loads(text)
        d["cells"] = [EvalCell(**c) for c in d["cells"]]
        return cls(**d)

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(["obs_size", "trained_rand_shape", "eval_rand_shape", "width", "episodes", "mean", "std"])
        for c in self.cells:
            w.writerow([c.obs_size, int(c.trained_rand_shape), int(c.eval_rand_shape), c.width, c.episodes,
                        repr(c.mean), repr(c.std)])
        return buf.getvalue()

    @classmethod
    def from_csv(cls, text: str, *, domain: str = "", checkpoint_step: int = 0) -> "EvalReport":
        cells = [EvalCell(obs_size=int(r["obs_size"]), trained_rand_shape=bool(int(r["trained_rand_shape"])),
                          eval_rand_shape=bool(int(r["eval_rand_shape"])), width=int(r["width"]),
                          episodes=int(r["episodes"]), mean=float(r["mean"]), std=float(r["std"]))
                 for r in csv.DictReader(io.StringIO(text))]
        return cls(domain=domain, checkpoint_step=checkpoint_step, n_seeds=0, episodes_per_seed=0, cells=cells)


def _cell_env_seed(base_seed: int, cell_idx: int, seed_idx: int) -> int:
    """harness._cell_env_seed (harness.py:271-273)."""
    ss = np.random.SeedSequence(entropy=base_seed, spawn_key=(cell_idx, seed_idx))
    return int(ss.generate_state(1, np.uint64)[0])


def env_config_from_dict(d: dict) -> EnvConfig:
    """ppo.env_config_from_dict (ppo.py:371-376)."""
    d = dict(d)
    for key in ("pinpoints", "controllable"):
        if key in d and d[key] is not None:
            d[key] = tuple(d[key])
    return EnvConfig(**d)


def evaluate(checkpoint, *, widths: Sequence[int] = EVAL_WIDTHS, eval_shapes: Sequence[bool] = (False, True),
             n_seeds: int = 3, episodes_per_seed: int = 32, seed: int = 0, greedy: bool = True, device=None,
             act_factory: Callable | None = None, check_every: int = 16) -> EvalReport:
    """The width x shape generalisation grid (harness.py:275-342) on the GPU.

    Each cell runs ``n_seeds`` batches of ``episodes_per_seed`` envs (seeded
    from (seed, cell index, seed index)) with ``deterministic_metrics=True``
    and the default episode length; mean and population std over all first
    episode rewards. ``act_factory(model, cell_seed)`` replaces the policy
    (tests use it to run a policy whose actions are exact integers).
    """
    from .policy import Checkpoint, load_checkpoint

    torch = _torch()
    if n_seeds < 1 or episodes_per_seed < 1:
        raise ValueError("need at least one seed and one episode")
    ck = checkpoint if isinstance(checkpoint, Checkpoint) else load_checkpoint(checkpoint)
    dev = torch.device(device if device is not None else "cuda")
    model = ck.build_model(dev)
    model.eval()
    base_cfg = env_config_from_dict(ck.meta["env"])
    if ck.arch.obs_size != base_cfg.obs_size:
        raise ValueError("checkpoint architecture and environment observation size disagree")
    cells = []
    cell_idx = 0
    for eval_rand in eval_shapes:
        for width in widths:
            cfg = replace(base_cfg, max_width=width, max_height=width, randomize_shape=bool(eval_rand),
                          deterministic_metrics=True, max_steps=None)
            rewards = []
            for seed_idx in range(n_seeds):
                cs = _cell_env_seed(seed, cell_idx, seed_idx)
                env = BatchEnv(cfg, episodes_per_seed, seed=cs, device=dev, validate=False)
                if act_factory is not None:
                    act = act_factory(model, cs)
                elif greedy:
                    act = greedy_policy(model)
                else:
                    sampler = torch.Generator(device=dev)
                    sampler.manual_seed(cs % (2 ** 63))
                    act = sampling_policy(model, sampler)
                rewards.append(first_episode_rewards(env, act, check_every=check_every))
            all_rewards = np.concatenate(rewards)
            cells.append(EvalCell(obs_size=base_cfg.obs_size, trained_rand_shape=base_cfg.randomize_shape,
                                  eval_rand_shape=bool(eval_rand), width=int(width), episodes=all_rewards.size,
                                  mean=float(all_rewards.mean()), std=float(all_rewards.std())))
            cell_idx += 1
    return EvalReport(domain=base_cfg.domain, checkpoint_step=ck.step, n_seeds=n_seeds,
                      episodes_per_seed=episodes_per_seed, cells=cells)


def random_baseline(env_config: EnvConfig, episodes: int = 1000, *, seed: int = 0, device=None,
                    check_every: int = 16) -> tuple[float, float]:
    """harness.random_baseline (harness.py:376-386): mean and population std of
    the first episode reward under uniform random actions (the reference's
    numpy stream ``default_rng(seed + 1)``, so the result is bit-identical)."""
    if episodes < 100:
        raise ValueError("need at least 100 episodes for a stable baseline")
    env = BatchEnv(env_config, episodes, seed=seed, device=device, validate=False)
    act = uniform_policy(env_config.n_actions, np.random.default_rng(seed + 1))
    rewards = first_episode_rewards(env, act, check_every=check_every)
    return float(rewards.mean()), float(rewards.std())


__all__ = ["first_episode_rewards", "greedy_policy", "sampling_policy", "uniform_policy", "BenchRow",
           "BenchReport", "bench_random_fps", "EvalCell", "EvalReport", "evaluate", "random_baseline",
           "env_config_from_dict", "EVAL_WIDTHS", "BENCH_LADDER"]
