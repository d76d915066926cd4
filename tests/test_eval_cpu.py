"""Eval-path host logic and its golden fixtures, without a GPU.

``tests/golden/eval.npz`` comes from the live reference harness
(``tests/golden/make_eval_golden.py``). Here the CPU oracle reproduces its
``first_episode_rewards`` under ``uniform_policy`` (harness.py:48-61,83-87)
bit-exactly, which pins the fixture and the oracle to each other; the device
path is compared with the same fixture in ``tests/test_gpu_eval.py``.
"""
import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_2408_12525_b200.config import EnvConfig
from paper_2408_12525_b200.harness import EvalReport, _cell_env_seed
from tests._golden import load

Z = load("eval.npz")
CASES = sorted({k.split("_")[1] if k.count("_") == 2 else "_".join(k.split("_")[1:-1])
                for k in Z.files if k.startswith("rb_") and k.endswith("_mean")})


def _cfg(name):
    kw = json.loads(str(Z[f"rb_{name}_config"]))
    for k in ("pinpoints", "controllable"):
        if k in kw:
            kw[k] = tuple(kw[k])
    return EnvConfig(**kw)


def oracle_first_episode_rewards(cfg, n, seed):
    env = O.OracleBatchEnv(cfg, n, seed=seed)
    env.reset()
    rng = np.random.default_rng(seed + 1)
    rewards = np.zeros(n)
    seen = np.zeros(n, dtype=bool)
    while not seen.all():
        r, done, info = env.step_no_obs_info(rng.integers(0, cfg.n_actions, size=n))
        first = done & ~seen
        rewards[first] = info["episode_reward"][first]
        seen |= first
    return rewards


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_random_baseline(name):
    cfg = _cfg(name)
    n, seed = int(Z[f"rb_{name}_episodes"]), int(Z[f"rb_{name}_seed"])
    r = oracle_first_episode_rewards(cfg, n, seed)
    assert np.array_equal(r, Z[f"rb_{name}_rewards"])
    assert float(r.mean()) == float(Z[f"rb_{name}_mean"]) and float(r.std()) == float(Z[f"rb_{name}_std"])


def test_eval_report_encodings_round_trip():
    rep = EvalReport.from_json(str(Z["eval_greedy_json"]))
    assert EvalReport.from_json(rep.to_json()) == rep
    back = EvalReport.from_csv(rep.to_csv(), domain=rep.domain, checkpoint_step=rep.checkpoint_step)
    assert back.cells == rep.cells


def test_cell_seeds_follow_the_reference():
    # harness._cell_env_seed (harness.py:271-273)
    ss = np.random.SeedSequence(entropy=5, spawn_key=(3, 1))
    assert _cell_env_seed(5, 3, 1) == int(ss.generate_state(1, np.uint64)[0])
