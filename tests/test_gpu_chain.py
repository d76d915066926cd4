"""lg_step_random: chained (programmatic dependent) step launches.

``BatchEnv.step_random(seed, ...)`` draws each env's action in the step
kernel -- the values ``random_actions(seed)`` writes -- and steps; consecutive
calls overlap launch to launch (env_kernels.cuh chain_enter/chain_leave).
Parity bar: bit-identical to ``random_actions`` + ``step_raw`` (itself pinned
to the oracle by test_gpu_parity.py), through episodes with auto-resets, for
the solo warp/block kernels and the lane-team kernels, eagerly and in a CUDA
graph, with no reads between the chained launches.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

CASES = [
    # (config, envs, steps): multi-wave solo warp mode (c5 shape), episodes end
    (dict(domain="binary", max_steps=20), 131_072 + 77, 45),
    # small batch (lane team 16 by default) and the dungeon spec kernel (c3 shape)
    (dict(domain="binary", max_steps=7), 300, 20),
    (dict(domain="dungeon", representation="wide", randomize_shape=True, change_budget=9, max_steps=30),
     65_536, 40),
    # lane teams: G16 maze turtle (c2 spec) and G64 binary (c4 spec)
    (dict(domain="maze", representation="turtle", max_width=16, max_height=16, obs_size=31, max_steps=25),
     4_096 + 5, 40),
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7, max_steps=12), 2_000, 20),  # unchained
    (dict(domain="dungeon", max_width=32, max_height=24, obs_size=15, max_steps=10), 3_000, 20),  # G32
    # generic kernels: control planes + pinpoints
    (dict(domain="maze", pinpoints=("player", "door"), controllable=("path_length",), max_steps=15),
     5_000, 20),
]


def _same_state(a, b, path=""):
    if isinstance(a, dict):
        assert a.keys() == b.keys(), path
        for k in a:
            _same_state(a[k], b[k], f"{path}/{k}")
    elif isinstance(a, np.ndarray):
        assert np.array_equal(a, b), path
    else:
        assert a == b, path


def _buffers(env):
    B, dev = env.n_envs, env.device
    return dict(obs=env.new_obs(), reward=torch.empty(B, dtype=torch.float64, device=dev),
                done=torch.empty(B, dtype=torch.bool, device=dev), info=env._info_buffers(),
                stats=torch.zeros(5, dtype=torch.float64, device=dev),
                acts=torch.empty(B, dtype=torch.int64, device=dev))


def _pair(kw, n):
    cfg = EnvConfig(**kw)
    a = BatchEnv(cfg, n, seed=3, validate=False)
    b = BatchEnv(cfg, n, seed=3, validate=False)
    ba, bb = _buffers(a), _buffers(b)
    a.reset(out=ba["obs"])
    b.reset(out=bb["obs"])
    return a, b, ba, bb


def _seq_step(env, buf, seed):
    env.random_actions(seed, out=buf["acts"])
    env.step_raw(buf["acts"], buf["obs"], buf["reward"], buf["done"], buf["info"], buf["stats"])


def _chain_step(env, buf, seed):
    env.step_random(seed, buf["obs"], buf["reward"], buf["done"], buf["info"], buf["stats"],
                    actions_out=buf["acts"])


def _compare(a, b, ba, bb):
    torch.cuda.synchronize()
    for k in ("obs", "reward", "done", "acts"):
        assert torch.equal(ba[k], bb[k]), k
    for k in ba["info"]:
        assert torch.equal(ba["info"][k], bb["info"][k]), k
    # episode stats: same episodes (atomic float sums: order-free count, close sums)
    assert float(ba["stats"][0]) == float(bb["stats"][0])
    assert torch.allclose(ba["stats"], bb["stats"], rtol=1e-12, atol=1e-9)
    _same_state(a.state_dict(), b.state_dict())
    assert a.errors() == 0 and b.errors() == 0


@pytest.mark.parametrize("case", range(len(CASES)))
def test_chained_steps_equal_random_actions_plus_step(case):
    kw, n, steps = CASES[case]
    a, b, ba, bb = _pair(kw, n)
    for i in range(steps):  # no reads between the chained launches
        _chain_step(a, ba, 1000 + i)
        _seq_step(b, bb, 1000 + i)
    _compare(a, b, ba, bb)
    assert float(ba["stats"][0]) > 0  # episodes ended (auto-resets inside the chain)


@pytest.mark.parametrize("case", [0, 2, 3])
def test_chained_steps_in_a_cuda_graph(case):
    kw, n, steps = CASES[case]
    a, b, ba, bb = _pair(kw, n)
    K = 8
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            _chain_step(a, ba, 500 + i)
    for rep in range(3):  # each replay: the same K seeds
        g.replay()
        for i in range(K):
            _seq_step(b, bb, 500 + i)
    _compare(a, b, ba, bb)


def test_chain_interleaved_with_other_calls():
    """A chain broken by other calls on the env (step, observe, state
    export) restarts with a plain launch and stays exact."""
    kw, n, _ = CASES[0]
    a, b, ba, bb = _pair(kw, n)
    for i in range(30):
        if i % 7 == 3:
            b.random_actions(77 + i, out=bb["acts"])
            ba["acts"].copy_(bb["acts"])
            a.step_raw(ba["acts"], ba["obs"], ba["reward"], ba["done"], ba["info"], ba["stats"])
            b.step_raw(bb["acts"], bb["obs"], bb["reward"], bb["done"], bb["info"], bb["stats"])
        elif i % 7 == 5:
            a.observe(out=ba["obs"])
            a.state_dict()
            _seq_step(b, bb, 77 + i)
            _chain_step(a, ba, 77 + i)
        else:
            _chain_step(a, ba, 77 + i)
            _seq_step(b, bb, 77 + i)
    _compare(a, b, ba, bb)


def test_chained_solo_block_mode(monkeypatch):
    """Small batches default to lane teams; the solo block-mode kernel chained."""
    monkeypatch.setenv("LG_SOLO_SMALL", "1")
    test_chained_steps_equal_random_actions_plus_step(1)


def test_chain_disabled_by_env(monkeypatch):
    monkeypatch.setenv("LG_NO_CHAIN", "1")
    kw, n, steps = CASES[0]
    a, b, ba, bb = _pair(kw, n)
    for i in range(10):
        _chain_step(a, ba, i)
        _seq_step(b, bb, i)
    _compare(a, b, ba, bb)


@pytest.mark.parametrize("case", [0, 1, 3, 4, 5])
def test_episode_stats_are_the_finished_episodes(case):
    """lg_step's `stats` (block-aggregated counters, env_kernels.cuh
    block_stats_*) equal the sums over the envs whose info reports a
    finished episode, step after step, through lockstep resets."""
    kw, n, steps = CASES[case]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=9, validate=False)
    b = _buffers(env)
    env.reset(out=b["obs"])
    want = torch.zeros(5, dtype=torch.float64, device="cuda")
    for i in range(steps):
        env.random_actions(40 + i, out=b["acts"])
        env.step_raw(b["acts"], b["obs"], b["reward"], b["done"], b["info"], b["stats"])
        d = b["info"]["terminal"]
        want[0] += d.sum()
        want[1] += b["info"]["episode_reward"][d].sum()
        want[2] += b["info"]["episode_length"][d].double().sum()
        want[3] += b["info"]["episode_start_loss"][d].sum()
        want[4] += b["info"]["final_loss"][d].sum()
    torch.cuda.synchronize()
    assert float(want[0]) > 0
    assert float(b["stats"][0]) == float(want[0]) and float(b["stats"][2]) == float(want[2])
    assert torch.allclose(b["stats"], want, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("obs_dtype", ["uint8", "bits"])
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_chained_steps_other_observation_formats(case, obs_dtype):
    """uint8 planes and the packed bit stream (chained unless the stream has
    words shared between blocks, which need a memset before each step)."""
    kw, n, steps = CASES[case]
    cfg = EnvConfig(**kw)
    a = BatchEnv(cfg, n, seed=3, validate=False, obs_dtype=obs_dtype)
    b = BatchEnv(cfg, n, seed=3, validate=False, obs_dtype=obs_dtype)
    ba, bb = _buffers(a), _buffers(b)
    a.reset(out=ba["obs"])
    b.reset(out=bb["obs"])
    for i in range(min(steps, 25)):
        _chain_step(a, ba, 300 + i)
        _seq_step(b, bb, 300 + i)
    _compare(a, b, ba, bb)


def test_step_random_argument_checks():
    cfg = EnvConfig(domain="binary", max_width=8, max_height=8, obs_size=5)
    env = BatchEnv(cfg, 40, seed=0, validate=False)
    b = _buffers(env)
    with pytest.raises(RuntimeError):
        _chain_step(env, b, 0)
    env.reset(out=b["obs"])
    with pytest.raises(ValueError):
        env.step_random(0, b["obs"], b["reward"].float(), b["done"])
    with pytest.raises(ValueError):
        env.step_random(0, b["obs"][:20], b["reward"], b["done"])
    with pytest.raises(ValueError):
        env.step_random(0, b["obs"], b["reward"], b["done"], actions_out=b["acts"].int())
    _chain_step(env, b, 0)
    assert env.errors() == 0


@pytest.mark.parametrize("seed", range(24))
def test_chained_random_config_fuzz(seed):
    """Random configs (test_gpu_parity._random_config) and batch sizes that
    reach every kernel family: the chained path equals the unchained one."""
    from tests.test_gpu_parity import _random_config
    rng = np.random.default_rng(7000 + seed)
    cfg = _random_config(rng)
    n = int(rng.choice([37, 300, 4096 + 3, 20000, 40001]))
    try:
        a = BatchEnv(cfg, n, seed=seed, validate=False)
        b = BatchEnv(cfg, n, seed=seed, validate=False)
    except ValueError:
        pytest.skip("config rejected on device (limits)")
    ba, bb = _buffers(a), _buffers(b)
    a.reset(out=ba["obs"])
    b.reset(out=bb["obs"])
    if a.errors() or b.errors():
        pytest.skip("reset flagged (pinpoints do not fit)")
    for i in range(30):
        _chain_step(a, ba, 50 + i)
        _seq_step(b, bb, 50 + i)
    torch.cuda.synchronize()
    for k in ("obs", "reward", "done", "acts"):
        assert torch.equal(ba[k], bb[k]), k
    for k in ba["info"]:
        assert torch.equal(ba["info"][k], bb["info"][k]), k
    _same_state(a.state_dict(), b.state_dict())
    assert a.errors() == b.errors()


@pytest.mark.parametrize("n", [1, 300, 20000])
def test_chained_steps_without_observations(n):
    """obs=None (no observation written), down to a single env."""
    cfg = EnvConfig(domain="maze", representation="turtle", max_steps=9)
    a, b, ba, bb = _pair(dict(domain="maze", representation="turtle", max_steps=9), n)
    for i in range(20):
        a.step_random(900 + i, None, ba["reward"], ba["done"], ba["info"], ba["stats"], actions_out=ba["acts"])
        b.random_actions(900 + i, out=bb["acts"])
        b.step_raw(bb["acts"], None, bb["reward"], bb["done"], bb["info"], bb["stats"])
    torch.cuda.synchronize()
    for k in ("reward", "done", "acts"):
        assert torch.equal(ba[k], bb[k]), k
    _same_state(a.state_dict(), b.state_dict())
    assert cfg.n_actions == 8
