"""BASELINE.json's five configs at their stated sizes, through full episodes,
against the CPU oracle (needs a B200).

Every config runs at the batch size BASELINE.json names. c1-c4 are compared
env for env with an oracle batch of the same size; c5 (2^20 envs) is compared
on two 4,096-env slices, which the oracle reproduces from the same global
stream indices (``OracleBatchEnv(offset=lo)``, reference spawn_rngs
env.py:591-594). Episode lengths are 3*h*w (env.py:292), so c1/c2/c5 run past
step 768, where every env of the lockstep batch auto-resets at once
(env.py:391-392), and c3's random shapes (3..16 per side) reset many times.

Rewards, dones and the info dict are compared on every step, bit-exactly
(float64 rewards reproduce the reference's canonical-order arithmetic; the
north-star tolerance, 1e-6 relative, is asserted as well); observations every
``obs_every`` steps and at the end; the final state (maps, metrics, counters,
PCG64 states) at the end.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import INFO_KEYS, BatchEnv  # noqa: E402

pytestmark = pytest.mark.gpu
REL_TOL = 1e-6

# name -> (EnvConfig kwargs, n_envs, steps, obs_every); BASELINE.json configs[0..3]
FULL = {
    "c1": (dict(domain="binary"), 64, 800, 1),
    "c2": (dict(domain="maze", representation="turtle"), 4096, 800, 25),
    "c3": (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
                randomize_shape=True), 65536, 60, 10),
    "c4": (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 65536, 12, 3),
}
STATE_KEYS = ("tiles", "active", "frozen", "shape_hw", "order_len", "pos_idx", "pos", "t", "changes",
              "max_steps", "lo", "hi", "values", "unreach", "prev_loss", "ep_reward", "ep_start_loss",
              "rng")


def _np(x):
    return x.detach().cpu().numpy()


def _cmp_step(t, got, want, sl=slice(None)):
    o1, r1, d1, i1 = got
    o2, r2, d2, i2 = want
    r1 = _np(r1[sl])
    assert np.array_equal(r1, r2), (t, np.flatnonzero(r1 != r2)[:8])
    assert np.allclose(r1, r2, rtol=REL_TOL, atol=0)
    assert np.array_equal(_np(d1[sl]), d2), t
    for k in INFO_KEYS:
        assert np.array_equal(_np(i1[k][sl]), i2[k]), (k, t)


@pytest.mark.parametrize("name", sorted(FULL))
def test_baseline_config_full_size(name):
    kw, n, steps, obs_every = FULL[name]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=0, validate=False)
    ref = O.OracleBatchEnv(cfg, n, seed=0)
    assert np.array_equal(_np(env.reset()), ref.reset())
    act = np.random.default_rng(n)  # the harness convention (harness.py:165)
    ends = 0
    for t in range(steps):
        a = act.integers(0, cfg.n_actions, size=n)
        want_obs = (t + 1) % obs_every == 0 or t == steps - 1
        got = env.step(torch.from_numpy(a).cuda())
        if want_obs:
            want = ref.step(a)
        else:
            want = (None,) + tuple(ref.step_no_obs_info(a))
        _cmp_step(t, got, want)
        if want_obs:
            assert np.array_equal(_np(got[0]), want[0]), (name, t)
        ends += int(want[2].sum())
    if name != "c4":  # c4's episodes are 3*64*64 = 12,288 steps; its reset path is pinned by
        assert ends > 0, "the run must cover auto-resets"  # test_gpu_parity's 64x40 budget case
    s1, s2 = env.state_dict(), ref.state_dict()
    for k in STATE_KEYS:
        assert np.array_equal(s1[k], s2[k]), (name, k)
    assert env.errors() == 0


def test_baseline_c5_full_size_slices():
    """c5: 2^20 envs on the GPU; two 4,096-env slices (one unaligned to warps
    and blocks, one at the ragged end) replayed by the oracle from the same
    global stream indices and the same per-env device actions, for 800 steps
    (the lockstep auto-reset of every env happens at step 768)."""
    cfg = EnvConfig(domain="binary")
    n, cnt, steps = 1 << 20, 4096, 800
    slices = [123_457, n - cnt]
    env = BatchEnv(cfg, n, seed=0, validate=False)
    refs = [O.OracleBatchEnv(cfg, cnt, seed=0, offset=lo) for lo in slices]
    obs = env.reset()
    for lo, ref in zip(slices, refs):
        assert np.array_equal(_np(obs[lo:lo + cnt]), ref.reset())
    acts = torch.empty(n, dtype=torch.int64, device="cuda")
    ends = 0
    for t in range(steps):
        env.random_actions(7919 * t + 1, out=acts)
        got = env.step(acts)
        a_host = _np(acts)
        check_obs = (t + 1) % 50 == 0 or t in (766, 767, 768) or t == steps - 1
        for lo, ref in zip(slices, refs):
            sl = slice(lo, lo + cnt)
            a = a_host[sl]
            if check_obs:
                want = ref.step(a)
                assert np.array_equal(_np(got[0][sl]), want[0]), (lo, t)
            else:
                want = (None,) + tuple(ref.step_no_obs_info(a))
            _cmp_step(t, got, want, sl)
            ends += int(want[2].sum())
    assert ends == 2 * cnt, ends  # every env of both slices finished exactly one episode (t = 768)
    sd = env.state_dict()
    for lo, ref in zip(slices, refs):
        s2 = ref.state_dict()
        for k in ("tiles", "frozen", "pos_idx", "t", "changes", "prev_loss", "ep_reward", "rng"):
            assert np.array_equal(sd[k][lo:lo + cnt], s2[k]), (lo, k)
        for k in ("values", "unreach", "lo", "hi"):
            assert np.array_equal(sd[k][:, lo:lo + cnt], s2[k]), (lo, k)
    assert env.errors() == 0
