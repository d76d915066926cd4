"""Pin the CPU oracle to the live reference (fixtures from tests/golden/make_golden.py)
and to the SURVEY.md Appendix C digests. CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2408_12525_b200.config import EnvConfig
from tests._golden import digest, env_case_names, load, load_env_case


def test_rng_spawn_and_plain_states():
    z = load("rng.npz")
    for seed in (0, 7, 123456789, 2 ** 40 + 3):
        idx = z[f"spawn_{seed}_idx"]
        want = z[f"spawn_{seed}_states"]
        for k, i in enumerate(idx):
            got = O.seed_streams(seed, int(i), 1)[0]
            assert np.array_equal(got[:4], want[k]), (seed, i)
        assert np.array_equal(O.seed_plain(seed)[:4], z[f"plain_{seed}_state"])


def test_rng_draw_sequences():
    z = load("rng.npz")
    bounds = [1, 2, 3, 7, 100, 257, 4097, 2 ** 31 + 5]
    for seed in (0, 7, 123456789, 2 ** 40 + 3):
        g = O.seed_plain(seed)
        got = []
        for k in range(400):
            got.append(int(O.rng_draw(g, 3, 1, bounds[k % 8])[0]))
            got.append(int(O.rng_draw(g, 3, 1, 2 ** 63)[0]))
            got.append(int(O.rng_draw(g, 2, 1)[0]))
        assert np.array_equal(np.array(got, dtype=np.uint64), z[f"draws_{seed}"]), seed
        ch = []
        for k in range(100):
            ch.extend(int(x) for x in O.rng_draw(g, 4, 1, 9 + 37 * k, 1 + k % 5))
        assert np.array_equal(np.array(ch, dtype=np.int64), z[f"choice_{seed}"]), seed


def test_metrics_against_reference():
    z = load("metrics.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files if k.endswith("_tiles") and not k.startswith("exh3")})
    assert len(keys) == 21
    for key in keys:
        domain = key.split("_")[0]
        tiles, active = z[f"{key}_tiles"], z[f"{key}_active"]
        rng = O.seed_streams(int(z[f"{key}_seed"]), 0, tiles.shape[0])
        vals, unr = O.metrics(domain, tiles, active, rng if domain == "binary" else None)
        assert np.array_equal(vals, z[f"{key}_values"]), key
        assert np.array_equal(unr, z[f"{key}_unreach"]), key


def test_metrics_exhaustive_3x3():
    z = load("metrics.npz")
    tiles = z["exh3_tiles"]
    vals, _ = O.metrics("binary", tiles, np.ones_like(tiles), O.seed_streams(3, 0, 512))
    assert np.array_equal(vals, z["exh3_values"])


@pytest.mark.parametrize("name", env_case_names())
def test_env_case(name):
    cfg, z = load_env_case(name)
    n, steps = int(z["n_envs"]), int(z["steps"])
    env = O.OracleBatchEnv(cfg, n, seed=int(z["seed"]))
    obs = env.reset()
    assert digest(obs) == str(z["obs_digests"][0])
    sd = env.state_dict()
    assert np.array_equal(sd["tiles"], z["reset_tiles"])
    assert np.array_equal(sd["values"], z["reset_values"])
    assert np.array_equal(sd["prev_loss"], z["reset_prev_loss"])
    for t in range(steps):
        obs, r, d, info = env.step(z["actions"][t])
        assert np.array_equal(r, z["rewards"][t]), (name, t)
        assert np.array_equal(d, z["dones"][t]), (name, t)
        for k in ("episode_reward", "episode_length", "episode_start_loss", "final_loss"):
            assert np.array_equal(info[k], z[f"info_{k}"][t]), (name, k, t)
        assert digest(obs) == str(z["obs_digests"][t + 1]), (name, t)
    sd = env.state_dict()
    assert np.array_equal(sd["tiles"], z["final_tiles"])
    assert np.array_equal(sd["frozen"], z["final_frozen"])
    assert np.array_equal(sd["values"], z["final_values"])
    assert np.array_equal(sd["unreach"], z["final_unreach"])
    assert np.array_equal(sd["pos_idx"], z["final_pos_idx"])
    assert np.array_equal(sd["t"], z["final_t"])
    assert np.array_equal(sd["prev_loss"], z["final_prev_loss"])
    assert np.array_equal(sd["ep_reward"], z["final_ep_reward"])
    assert np.array_equal(sd["rng"], z["final_rng"])
    if cfg.representation != "wide":
        assert np.array_equal(sd["pos"], z["final_pos"])


# SURVEY.md Appendix C (numpy 2.3.5 live-oracle digests).
APPENDIX_C = [
    (dict(domain="binary"), 200, ("b66ea2f406f8c482", "455718836e4cf0cc", "59ec91dcb7dc65b5",
                                  "66f27c5db0420a57", "b4db42a3d4c7e283"), 16.0, 0),
    (dict(domain="binary"), 800, ("b66ea2f406f8c482", "54cca0188108d023", "cec2a02395560b61",
                                  "5bbffd418794b1f6", "29e8880bc159d43e"), 95.0, 64),
    (dict(domain="maze"), 200, ("9764442c0a8b0fd8", "434a79cd64c45307", "59ec91dcb7dc65b5",
                                "9fb92bee0424b57d", "b6211220ef0de296"), -4707.0, 0),
    (dict(domain="dungeon", pinpoints=("player", "key", "door"), randomize_shape=True), 200,
     ("f880a733ac647364", "3cfd2fdb1399afd0", "f9180636d4c4952b", "090ff05a5325ba77",
      "3253f631fbbbf450"), 3358.0, 23),
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 200,
     ("c913ff2def2f26e5", "43b1a6ccc57c8578", "59ec91dcb7dc65b5", "7abdbc395a5e527a",
      "99fad51ae8f77da1"), -47.0, 0),
]


@pytest.mark.parametrize("case", range(len(APPENDIX_C)))
def test_appendix_c_digests(case):
    kw, steps, want, rsum, ndone = APPENDIX_C[case]
    cfg = EnvConfig(**kw)
    n = 64
    env = O.OracleBatchEnv(cfg, n, seed=0)
    act = np.random.default_rng(n)
    obs = env.reset()
    sd = env.state_dict()
    got_reset = digest(sd["tiles"], sd["values"], sd["unreach"], obs)
    rewards, dones = [], []
    for _ in range(steps):
        obs, r, d, _ = env.step(act.integers(0, cfg.n_actions, size=n))
        rewards.append(r)
        dones.append(d)
    sd = env.state_dict()
    got = (got_reset, digest(*rewards), digest(*dones),
           digest(sd["tiles"], sd["values"], sd["unreach"], sd["pos_idx"], sd["t"]), digest(obs))
    assert got == want
    assert float(np.sum(rewards)) == rsum and int(np.sum(dones)) == ndone
