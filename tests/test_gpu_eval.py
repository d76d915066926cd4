"""The device eval path against the live reference harness (needs a B200).

Fixtures: ``tests/golden/eval.npz`` + the two checkpoints in the reference's
format, written by ``tests/golden/make_eval_golden.py`` from
``levelgen.harness`` (harness.py:48-87,275-342,376-386).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2408_12525_b200 import harness as H  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402
from tests._golden import GOLDEN, load  # noqa: E402
from tests.test_eval_cpu import CASES, _cfg  # noqa: E402

pytestmark = pytest.mark.gpu
Z = load("eval.npz")


@pytest.mark.parametrize("name", CASES)
def test_random_baseline_matches_reference(name):
    cfg = _cfg(name)
    n, seed = int(Z[f"rb_{name}_episodes"]), int(Z[f"rb_{name}_seed"])
    mean, std = H.random_baseline(cfg, n, seed=seed)
    assert mean == float(Z[f"rb_{name}_mean"]) and std == float(Z[f"rb_{name}_std"])


@pytest.mark.parametrize("check_every", [1, 7])
@pytest.mark.parametrize("name", CASES)
def test_first_episode_rewards_match_reference(name, check_every):
    cfg = _cfg(name)
    n, seed = int(Z[f"rb_{name}_episodes"]), int(Z[f"rb_{name}_seed"])
    env = BatchEnv(cfg, n, seed=seed)
    act = H.uniform_policy(cfg.n_actions, np.random.default_rng(seed + 1))
    r = H.first_episode_rewards(env, act, check_every=check_every)
    assert np.array_equal(r, Z[f"rb_{name}_rewards"])


def _hash_factory(n_actions):
    """tests/golden/make_eval_golden.py:hash_actions on device (exact int64)."""
    def factory(model, cell_seed):
        def act(obs):
            b = obs.shape[0]
            flat = (obs.reshape(b, -1) > 0.5).to(torch.int64)
            w = (torch.arange(flat.shape[1], dtype=torch.int64, device=obs.device) * 2654435761) % 1000003
            return (flat * w).sum(1) % n_actions
        return act
    return factory


def test_evaluate_grid_matches_reference_with_exact_actions():
    grid = json.loads(str(Z["eval_grid"]))
    want = H.EvalReport.from_json(str(Z["eval_hash_json"]))
    ck = os.path.join(GOLDEN, "eval_ckpt_hash.npz")
    n_actions = EnvConfig(domain="binary").n_actions
    got = H.evaluate(ck, widths=tuple(grid["widths"]), eval_shapes=tuple(grid["eval_shapes"]),
                     n_seeds=grid["n_seeds"], episodes_per_seed=grid["episodes_per_seed"], seed=grid["seed"],
                     act_factory=_hash_factory(n_actions))
    assert got == want, (got.to_csv(), want.to_csv())


def test_evaluate_grid_matches_reference_greedy_policy():
    """The real greedy ConvPolicy (float32, TF32 off) on device vs the
    reference's CPU evaluation: every cell's mean and std equal."""
    grid = json.loads(str(Z["eval_grid"]))
    want = H.EvalReport.from_json(str(Z["eval_greedy_json"]))
    got = H.evaluate(os.path.join(GOLDEN, "eval_ckpt_greedy.npz"), widths=tuple(grid["widths"]),
                     eval_shapes=tuple(grid["eval_shapes"]), n_seeds=grid["n_seeds"],
                     episodes_per_seed=grid["episodes_per_seed"], seed=grid["seed"])
    assert got == want, (got.to_csv(), want.to_csv())


def test_bench_random_fps_ladder():
    rep = H.bench_random_fps("binary", env_counts=(1, 64), seconds=0.2)
    assert [r.n_envs for r in rep.rows] == [1, 64] and all(r.fps > 0 for r in rep.rows)
    assert H.BenchReport.from_json(rep.to_json()).rows == rep.rows
