"""Golden fixtures for the evaluation path, from the LIVE reference harness.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_eval_golden.py

Writes ``eval.npz`` (+ ``eval_ckpt_*.npz`` checkpoints in the reference's own
format) next to this file:

* ``random_baseline`` (harness.py:376-386) and the per-env rewards of
  ``first_episode_rewards`` (harness.py:48-61) under ``uniform_policy``
  (harness.py:83-87) for three configs -- bit-exact targets;
* ``evaluate`` (harness.py:275-342) over a 2x2 width x shape grid with the
  action function replaced by ``hash_actions`` (an exact integer function of
  the observation, so the device run is bit-exact too);
* ``evaluate`` with the real greedy ConvPolicy (harness.py:64-70) of a
  checkpoint whose policy-head weights are scaled by 1e3, so argmax ties
  between float32 logits computed on different hardware are vanishingly rare.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import torch  # noqa: E402
from levelgen import harness as Hn  # noqa: E402
from levelgen import nets as N  # noqa: E402
from levelgen.env import BatchEnv, EnvConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

BASELINE_CASES = [
    ("binary8", dict(domain="binary", max_width=8, max_height=8, obs_size=7), 128, 3),
    ("dungeon16_pins_rand", dict(domain="dungeon", pinpoints=["player", "key", "door"], randomize_shape=True),
     100, 1),
    ("maze12x10_ctrl", dict(domain="maze", max_width=12, max_height=10, obs_size=9,
                            controllable=["path_length"]), 100, 2),
]
EVAL_ENV = dict(domain="binary", max_width=8, max_height=8, obs_size=9)
EVAL_GRID = dict(widths=(8, 12), eval_shapes=(False, True), n_seeds=2, episodes_per_seed=8, seed=5)


def hash_actions(obs: np.ndarray, n_actions: int) -> np.ndarray:
    """An exact integer function of a 0/1 observation (tests/test_gpu_eval.py
    computes the same on device)."""
    b = obs.shape[0]
    flat = (obs.reshape(b, -1) > 0.5).astype(np.int64)
    w = (np.arange(flat.shape[1], dtype=np.int64) * 2654435761) % 1000003
    return (flat @ w) % n_actions


def cfg_of(kw) -> EnvConfig:
    kw = dict(kw)
    for k in ("pinpoints", "controllable"):
        if k in kw:
            kw[k] = tuple(kw[k])
    return EnvConfig(**kw)


def main():
    out = {}
    for name, kw, episodes, seed in BASELINE_CASES:
        cfg = cfg_of(kw)
        mean, std = Hn.random_baseline(cfg, episodes, seed=seed)
        env = BatchEnv(cfg, episodes, seed=seed)
        rewards = Hn.first_episode_rewards(env, Hn.uniform_policy(cfg.n_actions, np.random.default_rng(seed + 1)))
        out[f"rb_{name}_config"] = np.array(json.dumps(kw))
        out[f"rb_{name}_episodes"] = np.array(episodes)
        out[f"rb_{name}_seed"] = np.array(seed)
        out[f"rb_{name}_mean"] = np.array(mean)
        out[f"rb_{name}_std"] = np.array(std)
        out[f"rb_{name}_rewards"] = rewards
        print(name, mean, std)

    cfg = cfg_of(EVAL_ENV)
    C = cfg.observation_shape[0] if hasattr(cfg, "observation_shape") else None
    env = BatchEnv(cfg, 1, seed=0)
    C = env.observation_shape[0]
    arch = N.default_arch(cfg.obs_size, C, cfg.n_actions)

    # (a) the grid machinery with an exact integer action function
    model = N.init_policy(arch, seed=0)
    path_a = os.path.join(OUT, "eval_ckpt_hash.npz")
    N.save_checkpoint(path_a, model, env_config=dict(EVAL_ENV), step=7)
    orig = Hn.greedy_policy
    Hn.greedy_policy = lambda m: (lambda obs: hash_actions(obs, cfg.n_actions))
    try:
        rep = Hn.evaluate(path_a, **EVAL_GRID)
    finally:
        Hn.greedy_policy = orig
    out["eval_hash_json"] = np.array(rep.to_json())
    print(rep.to_csv())

    # (b) the real greedy policy, head scaled so argmax is robust across hardware
    model = N.init_policy(arch, seed=1)
    with torch.no_grad():
        model.policy_head.weight.mul_(1000.0)
    path_b = os.path.join(OUT, "eval_ckpt_greedy.npz")
    N.save_checkpoint(path_b, model, env_config=dict(EVAL_ENV), step=11)
    rep = Hn.evaluate(path_b, **EVAL_GRID)
    out["eval_greedy_json"] = np.array(rep.to_json())
    out["eval_grid"] = np.array(json.dumps(EVAL_GRID))
    print(rep.to_csv())
    np.savez_compressed(os.path.join(OUT, "eval.npz"), **out)


if __name__ == "__main__":
    main()
