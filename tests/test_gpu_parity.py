"""CUDA path vs the oracle and the reference's golden fixtures (needs a B200).

Integer/byte outputs (maps, metrics, done flags, observations, RNG states) are
compared bit-exactly; rewards and losses are float64 and are compared
bit-exactly as well (the north-star tolerance is 1e-6 relative; the kernels
reproduce the reference's canonical-order float64 arithmetic exactly).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2408_12525_b200 import _lib  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv, NumpyBatchEnv  # noqa: E402
from tests._golden import digest, env_case_names, load, load_env_case  # noqa: E402

pytestmark = pytest.mark.gpu
REL_TOL = 1e-6  # north_star reward tolerance; bit-exact is asserted where it holds


def _np(x):
    return x.detach().cpu().numpy()


def _cmp_state(sd, want, prefix, rep):
    assert np.array_equal(sd["tiles"], want[f"{prefix}tiles"])
    assert np.array_equal(sd["frozen"], want[f"{prefix}frozen"])
    assert np.array_equal(sd["values"], want[f"{prefix}values"])
    assert np.array_equal(sd["unreach"], want[f"{prefix}unreach"])
    assert np.array_equal(sd["prev_loss"], want[f"{prefix}prev_loss"])


SMALL_CASES = ["c1_binary16_narrow_o31", "c2_maze16_turtle_o31", "c3_dungeon16_wide_pins_rand",
               "dungeon6_c5_like", "maze_ctrl_weights", "binary_ctrl_det_budget"]


@pytest.mark.parametrize("name", SMALL_CASES)
def test_golden_env_case_generic_kernels(name, monkeypatch):
    """The generic (runtime-flag) kernels on the cases the default launch
    sends to a specialised kernel (env_kernels.cuh spec_of)."""
    monkeypatch.setenv("LG_NO_SPEC", "1")
    test_golden_env_case(name)


@pytest.mark.parametrize("name", SMALL_CASES)
def test_golden_env_case_solo_block_path(name, monkeypatch):
    """Small batches on maps <= 16x16 run on 16-lane teams by default; keep
    them on the solo kernel (block mode) so both code paths are pinned on
    the same fixtures."""
    monkeypatch.setenv("LG_SOLO_SMALL", "1")
    test_golden_env_case(name)


@pytest.mark.parametrize("name", env_case_names())
def test_golden_env_case(name):
    cfg, z = load_env_case(name)
    n, steps = int(z["n_envs"]), int(z["steps"])
    env = BatchEnv(cfg, n, seed=int(z["seed"]))
    obs = env.reset()
    assert digest(_np(obs)) == str(z["obs_digests"][0]), "reset obs"
    sd = env.state_dict()
    _cmp_state(sd, {k[6:]: z[k] for k in z.files if k.startswith("reset_")}, "", cfg.representation)
    for t in range(steps):
        obs, r, d, info = env.step(torch.from_numpy(z["actions"][t]).cuda())
        r, d = _np(r), _np(d)
        assert np.array_equal(r, z["rewards"][t]), (name, t, np.flatnonzero(r != z["rewards"][t]))
        assert np.array_equal(d, z["dones"][t]), (name, t)
        for k in ("episode_reward", "episode_length", "episode_start_loss", "final_loss"):
            assert np.array_equal(_np(info[k]), z[f"info_{k}"][t]), (name, k, t)
        assert digest(_np(obs)) == str(z["obs_digests"][t + 1]), (name, t)
    sd = env.state_dict()
    assert np.array_equal(sd["tiles"], z["final_tiles"])
    assert np.array_equal(sd["frozen"], z["final_frozen"])
    assert np.array_equal(sd["values"], z["final_values"])
    assert np.array_equal(sd["unreach"], z["final_unreach"])
    assert np.array_equal(sd["pos_idx"], z["final_pos_idx"])
    assert np.array_equal(sd["t"], z["final_t"])
    assert np.array_equal(sd["changes"], z["final_changes"])
    assert np.array_equal(sd["shape_hw"], z["final_shape_hw"])
    assert np.array_equal(sd["prev_loss"], z["final_prev_loss"])
    assert np.array_equal(sd["ep_reward"], z["final_ep_reward"])
    assert np.array_equal(sd["rng"], z["final_rng"])
    assert np.array_equal(sd["metric_seeds"], z["final_metric_seeds"])
    if cfg.representation != "wide":
        assert np.array_equal(sd["pos"], z["final_pos"])
    assert env.errors() == 0


def test_metrics_kernel_against_reference_fixtures():
    z = load("metrics.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in z.files if k.endswith("_tiles") and not k.startswith("exh3")})
    lib = _lib.load()
    import ctypes
    for key in keys:
        domain = key.split("_")[0]
        tiles = torch.from_numpy(z[f"{key}_tiles"]).cuda()
        active = torch.from_numpy(z[f"{key}_active"].astype(np.uint8)).cuda()
        n, H, W = tiles.shape
        M = z[f"{key}_values"].shape[0]
        rng = torch.from_numpy(O.seed_streams(int(z[f"{key}_seed"]), 0, n).view(np.int64)).cuda()
        vals = torch.zeros((M, n), dtype=torch.int64, device="cuda")
        unr = torch.zeros((M, n), dtype=torch.uint8, device="cuda")
        code = {"binary": 0, "maze": 1, "dungeon": 2}[domain]
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(lib.lg_metrics(code, H, W, n, p(tiles), p(active), p(rng), p(vals), p(unr), None))
        torch.cuda.synchronize()
        assert np.array_equal(_np(vals), z[f"{key}_values"]), key
        assert np.array_equal(_np(unr).astype(bool), z[f"{key}_unreach"]), key


LIVE_CASES = [
    (dict(domain="binary"), 1000, 60, 3),
    (dict(domain="maze", representation="turtle"), 1000, 60, 4),
    (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
          randomize_shape=True), 1000, 60, 5),
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 300, 40, 6),
    (dict(domain="dungeon", max_width=5, max_height=5, obs_size=4, randomize_shape=True,
          pinpoints=("player", "key", "door"), max_steps=20, change_budget=6,
          controllable=("pkd_path", "regions", "nearest_enemy"), deterministic_metrics=True),
     777, 120, 7),
    (dict(domain="maze", max_width=33, max_height=17, obs_size=65, init_mode="weighted",
          randomize_shape=True, controllable=("regions",)), 200, 40, 8),
    (dict(domain="binary", max_width=64, max_height=40, obs_size=128, randomize_shape=True,
          change_budget=30), 64, 60, 9),
]


@pytest.mark.parametrize("case", range(len(LIVE_CASES)))
def test_live_oracle_side_by_side(case):
    kw, n, steps, seed = LIVE_CASES[case]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=seed)
    ref = O.OracleBatchEnv(cfg, n, seed=seed)
    assert np.array_equal(_np(env.reset()), ref.reset())
    act = np.random.default_rng(seed + n)
    for t in range(steps):
        a = act.integers(0, cfg.n_actions, size=n)
        o1, r1, d1, i1 = env.step(a)
        o2, r2, d2, i2 = ref.step(a)
        assert np.array_equal(_np(r1), r2), t
        assert np.allclose(_np(r1), r2, rtol=REL_TOL, atol=0)
        assert np.array_equal(_np(d1), d2), t
        for k in i2:
            assert np.array_equal(_np(i1[k]), i2[k]), (k, t)
        assert np.array_equal(_np(o1), o2), t
    s1, s2 = env.state_dict(), ref.state_dict()
    for k in ("tiles", "active", "frozen", "shape_hw", "order", "order_len", "pos_idx", "t", "changes",
              "max_steps", "lo", "hi", "values", "unreach", "prev_loss", "ep_reward", "ep_start_loss",
              "rng"):
        assert np.array_equal(s1[k], s2[k]), k


def test_sharded_batch_equals_unsharded():
    """global_offset shards reproduce the unsharded batch (multi-GPU partitioning)."""
    cfg = EnvConfig(domain="dungeon", pinpoints=("player", "key", "door"), randomize_shape=True)
    n = 512
    full = BatchEnv(cfg, n, seed=11)
    parts = [BatchEnv(cfg, 128, seed=11, global_offset=128 * k) for k in range(4)]
    of = _np(full.reset())
    op = np.concatenate([_np(p.reset()) for p in parts])
    assert np.array_equal(of, op)
    act = np.random.default_rng(0)
    for _ in range(50):
        a = act.integers(0, cfg.n_actions, size=n)
        of, rf, df, _ = full.step(a)
        outs = [p.step(a[128 * k:128 * (k + 1)]) for k, p in enumerate(parts)]
        assert np.array_equal(_np(of), np.concatenate([_np(o[0]) for o in outs]))
        assert np.array_equal(_np(rf), np.concatenate([_np(o[1]) for o in outs]))


def test_state_dict_round_trip_and_reference_format():
    cfg = EnvConfig(domain="maze", pinpoints=("player", "door"), controllable=("path_length",))
    env = BatchEnv(cfg, 300, seed=2)
    env.reset()
    act = np.random.default_rng(1)
    for _ in range(30):
        env.step(act.integers(0, cfg.n_actions, size=300))
    sd = env.state_dict()
    twin = BatchEnv(cfg, 300, seed=999)
    twin.load_state_dict(sd)
    ref = O.OracleBatchEnv(cfg, 300, seed=2)
    ref.reset()
    act = np.random.default_rng(1)
    for _ in range(30):
        ref.step(act.integers(0, cfg.n_actions, size=300))
    for _ in range(40):
        a = act.integers(0, cfg.n_actions, size=300)
        o1, r1, d1, _ = env.step(a)
        o2, r2, d2, _ = twin.step(a)
        o3, r3, d3, _ = ref.step(a)
        assert np.array_equal(_np(o1), _np(o2)) and np.array_equal(_np(o1), o3)
        assert np.array_equal(_np(r1), r3) and np.array_equal(_np(r2), r3)
    # reference-format rng_states round trip
    st = twin.state_dict()
    assert st["rng_states"][0]["bit_generator"] == "PCG64"
    g = np.random.Generator(np.random.PCG64())
    g.bit_generator.state = st["rng_states"][0]


@pytest.mark.parametrize("n", [16, 16384])
def test_numpy_facade_fresh_arrays_are_owned_by_the_caller(n):
    """copy=True returns new arrays every step (env.py:233) from recycled
    memory: arrays the caller keeps are never written again, released ones
    are reused, and every step's values equal the oracle's."""
    import gc
    cfg = EnvConfig(domain="binary", max_width=8, max_height=8, obs_size=5, max_steps=9)
    env = NumpyBatchEnv(cfg, n, seed=4)
    ref = O.OracleBatchEnv(cfg, n, seed=4)
    env.reset()
    ref.reset()
    act = np.random.default_rng(5)
    kept, want, addrs = [], [], set()
    for t in range(24):
        a = act.integers(0, cfg.n_actions, size=n)
        out = env.step(a)
        exp = ref.step(a)
        assert np.array_equal(out[0], exp[0]) and np.array_equal(out[1], exp[1]), t
        assert all(np.array_equal(out[3][k], exp[3][k]) for k in exp[3]), t
        if t % 3 == 0:  # keep every third step's arrays
            kept.append(out)
            want.append(exp)
        addrs.add(out[0].ctypes.data)
        del out
        gc.collect()
    for o, e in zip(kept, want):  # untouched by the later steps
        assert np.array_equal(o[0], e[0]) and np.array_equal(o[2], e[2])
        assert all(np.array_equal(o[3][k], e[3][k]) for k in e[3])
    assert len(addrs) < 24  # released arrays' memory was reused


def test_numpy_facade_and_errors():
    cfg = EnvConfig(domain="binary", max_width=8, max_height=8, obs_size=5)
    env = NumpyBatchEnv(cfg, 16, seed=1)
    with pytest.raises(RuntimeError):
        env.step(np.zeros(16, dtype=np.int64))
    ref = O.OracleBatchEnv(cfg, 16, seed=1)
    assert np.array_equal(env.reset(), ref.reset())
    with pytest.raises(ValueError):
        env.step(np.full(16, 3))
    with pytest.raises(ValueError):
        env.step(np.zeros(15, dtype=np.int64))
    act = np.random.default_rng(3)
    for _ in range(100):
        a = act.integers(0, cfg.n_actions, size=16)
        o1, r1, d1, i1 = env.step(a)
        o2, r2, d2, i2 = ref.step(a)
        assert np.array_equal(o1, o2) and np.array_equal(r1, r2) and np.array_equal(d1, d2)
        assert all(np.array_equal(i1[k], i2[k]) for k in i2)
    # device actions out of range: flagged, env takes a no-op step
    dev = BatchEnv(cfg, 4, seed=0, validate=False)
    dev.reset()
    dev.step(torch.tensor([0, 0, 7, 0], device="cuda"))
    assert dev.errors() & _lib.FLAG_BAD_ACTION
    assert dev.errors() == 0
    strict = BatchEnv(cfg, 4, seed=0)
    strict.reset()
    before = strict.state_dict()
    with pytest.raises(ValueError, match="out of range"):
        strict.step(torch.tensor([0, 0, 7, 0], device="cuda"))
    with pytest.raises(ValueError, match="out of range"):
        strict.step(torch.tensor([0, -1, 1, 0], device="cuda"))
    after = strict.state_dict()  # rejected before any mutation (env.py:358-361)
    for k in ("tiles", "pos_idx", "t", "changes", "prev_loss", "rng"):
        assert np.array_equal(before[k], after[k]), k
    twin = O.OracleBatchEnv(cfg, 4, seed=0)
    twin.reset()
    a = np.array([1, 2, 0, 1])
    o1, r1, _, _ = strict.step(torch.from_numpy(a).cuda())
    o2, r2, _, _ = twin.step(a)
    assert np.array_equal(_np(o1), o2) and np.array_equal(_np(r1), r2)


def test_validated_step_raises_auto_reset_errors():
    """An auto-reset that cannot place its pinpoints raises ValueError from
    the step (reset_rows -> place_pinpoints, grid.py:213-214), as the
    reference does; validate=False defers it to check_errors()."""
    cfg = EnvConfig(domain="maze", max_width=6, max_height=6, obs_size=5, randomize_shape=True,
                    pinpoints=("player",) * 10, max_steps=2)
    n = 4
    seed = next(s for s in range(100) if _resets_ok(cfg, n, s))
    for validate in (True, False):
        env = BatchEnv(cfg, n, seed=seed, validate=validate)
        ref = O.OracleBatchEnv(cfg, n, seed=seed)
        assert np.array_equal(_np(env.reset()), ref.reset())
        raised = False
        for t in range(400):
            a = np.zeros(n, dtype=np.int64)
            try:
                ref.step(a)
            except ValueError:
                raised = True
                if validate:
                    with pytest.raises(ValueError, match="pinpoints"):
                        env.step(a)
                else:
                    env.step(a)
                    with pytest.raises(ValueError, match="pinpoints"):
                        env.check_errors()
                break
            o1, r1, _, _ = env.step(a)
        assert raised


def _resets_ok(cfg, n, seed):
    try:
        O.OracleBatchEnv(cfg, n, seed=seed).reset()
        return True
    except ValueError:
        return False


def test_pinpoint_overflow_flags_error():
    cfg = EnvConfig(domain="maze", max_width=3, max_height=3, obs_size=3,
                    pinpoints=("player",) * 9)
    env = BatchEnv(cfg, 2)
    with pytest.raises(ValueError):
        env.reset()


WARP_MODE_CASES = [
    (dict(domain="binary"), 40000, 4),
    # episodes ending at different steps: warps mixing early-observation and
    # end-of-episode (auto-reset) envs, slot and stream layouts
    (dict(domain="binary", change_budget=2), 20000, 10),
    (dict(domain="dungeon", representation="wide", change_budget=3), 20000, 10),
    (dict(domain="maze", representation="turtle", max_steps=4), 19500, 9),
    (dict(domain="binary"), 19001, 4),  # ragged last warp and block
    (dict(domain="dungeon", representation="wide"), 18977, 3),  # ragged, stream layout
    (dict(domain="maze", representation="turtle"), 20000, 4),
    (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
          randomize_shape=True), 20000, 4),
    (dict(domain="maze", controllable=("path_length", "regions")), 20000, 3),
]


@pytest.mark.parametrize("layout", ["default", "stream", "slot", "generic"])
@pytest.mark.parametrize("case", range(len(WARP_MODE_CASES)))
def test_large_batch_warp_mode_against_oracle(case, layout, monkeypatch):
    """Batches >= 4 warps/SM take the warp-mode store path; pin it to the oracle
    with both shared-memory layouts (per-env slots, warp-wide bit stream), and
    the generic kernel (LG_NO_SPEC=1) where the default launch is specialised."""
    if layout == "generic":
        monkeypatch.setenv("LG_NO_SPEC", "1")
    elif layout != "default":
        monkeypatch.setenv("LG_STREAM", "1" if layout == "stream" else "0")
    kw, n, steps = WARP_MODE_CASES[case]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=21)
    ref = O.OracleBatchEnv(cfg, n, seed=21)
    assert np.array_equal(_np(env.reset()), ref.reset())
    act = np.random.default_rng(5)
    for t in range(steps):
        a = act.integers(0, cfg.n_actions, size=n)
        o1, r1, d1, _ = env.step(a)
        o2, r2, d2, _ = ref.step(a)
        assert np.array_equal(_np(r1), r2), t
        assert np.array_equal(_np(d1), d2), t
        assert np.array_equal(_np(o1), o2), t


@pytest.mark.parametrize("frozen_edit", [False, True])
def test_imported_frozen_cells_leave_the_fast_layout(frozen_edit, monkeypatch):
    """A no-pinpoint warp-mode batch skips the frozen plane (shared image and
    state reads) while every env's frozen plane is its border plane. Importing
    a state with active frozen cells (designer pins, load_state_dict) must
    switch back to the full layout: compare with the lane-team kernel, which
    always reads and renders the stored frozen plane."""
    cfg = EnvConfig(domain="binary", randomize_shape=True)
    n = 20000
    env = BatchEnv(cfg, n, seed=4)
    env.reset()
    act = np.random.default_rng(8)
    for _ in range(5):
        env.step(act.integers(0, cfg.n_actions, size=n))
    sd = env.state_dict()
    if frozen_edit:  # freeze active cells and redo the scan order as with_pin does
        from paper_2408_12525_b200.scalar import _scan_order, _serp_rank
        rng = np.random.default_rng(0)
        H, W = sd["tiles"].shape[1:]
        rank = _serp_rank(H, W)
        for b in rng.choice(n, size=500, replace=False):
            h, w = sd["shape_hw"][b]
            old = int(sd["order"][b, sd["pos_idx"][b]])
            sd["frozen"][b, rng.integers(h), rng.integers(w)] = True
            order = _scan_order(sd["active"][b], sd["frozen"][b])
            k = int(np.searchsorted(rank[order], rank[old])) % order.size
            sd["order"][b] = -1
            sd["order"][b, :order.size] = order
            sd["order_len"][b] = order.size
            sd["pos_idx"][b] = k
            sd["pos"][b] = divmod(int(order[k]), W)
    fast = BatchEnv(cfg, n, seed=0)
    fast.load_state_dict(sd)
    monkeypatch.setenv("LG_FORCE_TEAM", "1")
    team = BatchEnv(cfg, n, seed=0)
    team.load_state_dict(sd)
    assert np.array_equal(_np(fast.observe()), _np(team.observe()))
    for t in range(12):
        a = act.integers(0, cfg.n_actions, size=n)
        o1, r1, d1, _ = fast.step(a)
        o2, r2, d2, _ = team.step(a)
        assert np.array_equal(_np(r1), _np(r2)), t
        assert np.array_equal(_np(d1), _np(d2)), t
        assert np.array_equal(_np(o1), _np(o2)), t
    s1, s2 = fast.state_dict(), team.state_dict()
    for k in ("tiles", "frozen", "values", "prev_loss", "t"):
        assert np.array_equal(s1[k], s2[k]), k


def test_full_size_c5_properties():
    """2^20 envs (config c5): size-independent invariants of the outputs, and a
    shard built with global_offset reproduces its slice of the full batch."""
    cfg = EnvConfig(domain="binary")
    n = 1 << 20
    env = BatchEnv(cfg, n, seed=0, validate=False)
    obs = env.reset()
    for t in range(3):
        obs, r, d, info = env.step(env.random_actions(t))
    n_tiles = cfg.domain_obj.n_tiles
    one_hot = obs[:, : n_tiles + 1].sum(dim=1)
    assert bool((one_hot == 1.0).all())                       # tile planes are one-hot
    border, frozen = obs[:, n_tiles], obs[:, n_tiles + 1]
    assert bool((frozen >= border).all())                     # border cells read frozen
    assert bool((r == torch.round(r)).all())                  # unit weights: integer losses
    assert env.errors() == 0
    lo, cnt = 123456, 4096
    part = BatchEnv(cfg, cnt, seed=0, global_offset=lo, validate=False)
    part.reset()
    for t in range(3):
        # the same per-env actions the full batch received
        full_a = torch.empty(n, dtype=torch.int64, device="cuda")
        env2_a = env.random_actions(t, out=full_a)
        po, pr, _, _ = part.step(env2_a[lo:lo + cnt].contiguous())
    assert torch.equal(po, obs[lo:lo + cnt])
    assert torch.equal(pr, r[lo:lo + cnt])


def _random_config(rng):
    domain = ["binary", "maze", "dungeon"][int(rng.integers(3))]
    d = {"binary": ("diameter", "regions"),
         "maze": ("path_length", "regions", "n_player", "n_door"),
         "dungeon": ("pkd_path", "regions", "n_player", "n_key", "n_door", "n_enemy", "nearest_enemy")}[domain]
    piv = {"binary": (), "maze": ("player", "door"), "dungeon": ("player", "key", "door")}[domain]
    H, W = int(rng.integers(3, 65)), int(rng.integers(3, 65))
    if rng.random() < 0.5:
        H, W = int(rng.integers(3, 17)), int(rng.integers(3, 17))
    kw = dict(domain=domain, max_height=H, max_width=W,
              obs_size=int(rng.integers(3, min(128, 2 * max(H, W) - 1) + 1)),
              randomize_shape=bool(rng.random() < 0.5),
              representation=["narrow", "turtle", "wide"][int(rng.integers(3))],
              deterministic_metrics=bool(rng.random() < 0.3))
    if piv and rng.random() < 0.6:
        kw["pinpoints"] = tuple(rng.choice(piv, size=int(rng.integers(1, 4))))
    if rng.random() < 0.4:
        kw["controllable"] = tuple(sorted(set(rng.choice(d, size=int(rng.integers(1, 3))))))
    if rng.random() < 0.3:
        kw["init_mode"] = "weighted"
    if rng.random() < 0.3:
        kw["change_budget"] = int(rng.integers(1, 20))
    if rng.random() < 0.3:
        kw["max_steps"] = int(rng.integers(1, 60))
    if rng.random() < 0.3:
        kw["loss_weights"] = {m: float(rng.choice([0.5, 2.0, 0.25, 3.0])) for m in d[:2]}
    return EnvConfig(**kw)


@pytest.mark.parametrize("seed", range(64))
def test_random_config_fuzz_against_oracle(seed):
    """Random EnvConfigs (all domains/representations, 3..64 sides, windows up
    to 128, pins, controls, budgets, weights, deterministic metrics)."""
    rng = np.random.default_rng(1000 + seed)
    cfg = _random_config(rng)
    n = int(rng.integers(1, 300))
    env = BatchEnv(cfg, n, seed=seed)
    ref = O.OracleBatchEnv(cfg, n, seed=seed)
    try:
        o2 = ref.reset()
    except ValueError:
        with pytest.raises(ValueError):
            env.reset()
        return
    assert np.array_equal(_np(env.reset()), o2), cfg
    act = np.random.default_rng(seed)
    for t in range(40):
        a = act.integers(0, cfg.n_actions, size=n)
        try:
            o2, r2, d2, i2 = ref.step(a)
        except ValueError as exc:
            # an auto-reset that cannot place its pinpoints (grid.py:213-214):
            # the validated device step raises the same error on this step;
            # every earlier step was compared
            with pytest.raises(ValueError, match=str(exc).split(":")[0][:20]):
                env.step(a)
            return
        o1, r1, d1, i1 = env.step(a)
        assert np.array_equal(_np(r1), r2), (cfg, t)
        assert np.array_equal(_np(d1), d2), (cfg, t)
        assert np.array_equal(_np(o1), o2), (cfg, t)
    s1, s2 = env.state_dict(), ref.state_dict()
    for k in ("tiles", "frozen", "values", "unreach", "prev_loss", "rng", "t", "pos_idx"):
        assert np.array_equal(s1[k], s2[k]), (cfg, k)


U8_CASES = [
    (dict(domain="binary"), 40000, {}),                                   # solo warp, slot layout
    (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
          randomize_shape=True), 40000, {}),                              # solo warp, stream layout
    (dict(domain="binary"), 40000, {"LG_STREAM": "1"}),                   # stream layout, PE % 32 != 0
    (dict(domain="maze", representation="turtle"), 300, {"LG_SOLO_SMALL": "1"}),  # solo block mode
    (dict(domain="maze", representation="turtle"), 3000, {}),             # lane-team (mid-size)
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 500, {}),   # lane team 64
    (dict(domain="dungeon", max_width=40, max_height=20, obs_size=33), 257, {}),  # team 32, odd sizes
]


@pytest.mark.parametrize("case", range(len(U8_CASES)))
def test_uint8_observations_equal_float32(case, monkeypatch):
    kw, n, envs = U8_CASES[case]
    for k, v in envs.items():
        monkeypatch.setenv(k, v)
    cfg = EnvConfig(**kw)
    f32 = BatchEnv(cfg, n, seed=4)
    u8 = BatchEnv(cfg, n, seed=4, obs_dtype="uint8")
    a, b = f32.reset(), u8.reset()
    assert b.dtype == torch.uint8 and torch.equal(a.to(torch.uint8), b)
    for t in range(5):
        acts = f32.random_actions(t)
        a, ra, _, _ = f32.step(acts)
        b, rb, _, _ = u8.step(acts)
        assert torch.equal(a.to(torch.uint8), b) and torch.equal(ra, rb), t


def test_uint8_rejects_control_planes():
    with pytest.raises(ValueError):
        BatchEnv(EnvConfig(domain="maze", controllable=("path_length",)), 8, obs_dtype="uint8")


# Packed observation transfer (lg_step_host): the kernel writes the 0/1 planes
# as one bit stream, the host library expands it into the caller's array.
PACKED_CASES = [
    (dict(domain="binary"), 40000, {}),                                   # solo warp, slot + elided frozen plane
    (dict(domain="binary"), 19001, {}),                                   # ragged last warp
    (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
          randomize_shape=True), 20000, {}),                              # solo warp, stream layout
    (dict(domain="binary"), 20000, {"LG_STREAM": "1"}),                   # stream layout, PE % 32 != 0
    (dict(domain="binary"), 64, {"LG_SOLO_SMALL": "1"}),                  # block mode, shared words
    (dict(domain="maze", representation="turtle"), 300, {"LG_SOLO_SMALL": "1"}),  # block mode, E * PE % 32 != 0
    (dict(domain="binary"), 64, {}),                                      # c1: lane team 16
    (dict(domain="maze", representation="turtle"), 4096, {}),             # c2: lane team 16
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 500, {}),   # lane team 64 (c4 shape)
    (dict(domain="dungeon", max_width=40, max_height=20, obs_size=33), 257, {}),  # team 32, odd sizes
    (dict(domain="binary", max_width=8, max_height=8, obs_size=3), 37, {}),       # PE = 36 bits
    (dict(domain="maze", controllable=("path_length", "regions")), 500, {}),      # control planes: f32 copy
]


@pytest.mark.parametrize("obs_dtype", ["float32", "uint8"])
@pytest.mark.parametrize("case", range(len(PACKED_CASES)))
def test_packed_host_transfer_equals_device_obs(case, obs_dtype, monkeypatch):
    """NumpyBatchEnv.step (packed bits over PCIe, host expansion) returns the
    same observations as the device path, for every kernel and layout."""
    kw, n, envs = PACKED_CASES[case]
    monkeypatch.setenv("LG_HOST_EXPAND", "1")  # small batches would take the plain copy by default
    for k, v in envs.items():
        monkeypatch.setenv(k, v)
    cfg = EnvConfig(**kw)
    if obs_dtype == "uint8" and cfg.controllable:
        pytest.skip("uint8 observations exclude control planes")
    dev = BatchEnv(cfg, n, seed=9, obs_dtype=obs_dtype)
    host = NumpyBatchEnv(cfg, n, seed=9, obs_dtype=obs_dtype, pinned=(case % 2 == 0), copy=False)
    assert np.array_equal(_np(dev.reset()), host.reset())
    rng = np.random.default_rng(case)
    for t in range(4):
        a = rng.integers(0, cfg.n_actions, size=n)
        o1, r1, d1, i1 = dev.step(torch.from_numpy(a).cuda())
        o2, r2, d2, i2 = host.step(a)
        assert o2.dtype == np.dtype(obs_dtype)
        assert np.array_equal(_np(o1), o2), t
        assert np.array_equal(_np(r1), r2) and np.array_equal(_np(d1), d2), t
        assert all(np.array_equal(_np(i1[k]), i2[k]) for k in i2), t


def test_packed_and_float32_copy_paths_agree(monkeypatch):
    """LG_HOST_EXPAND=0 (float32 copy) and the packed path give equal arrays,
    including unaligned host buffers (numpy arrays offset by 4 bytes)."""
    cfg = EnvConfig(domain="binary")
    n = 1000
    a = NumpyBatchEnv(cfg, n, seed=2, copy=False)
    b = NumpyBatchEnv(cfg, n, seed=2, copy=False)
    a.reset()
    b.reset()
    rng = np.random.default_rng(0)
    for t in range(4):
        acts = rng.integers(0, cfg.n_actions, size=n)
        monkeypatch.setenv("LG_HOST_EXPAND", "0")
        o1 = a.step(acts)[0].copy()
        monkeypatch.setenv("LG_HOST_EXPAND", "1")
        o2 = b.step(acts)[0]
        assert np.array_equal(o1, o2), t
        if t == 1:  # from now on b expands into a 4-byte (not 16-byte) aligned array
            raw = np.empty(o2.nbytes + 16, dtype=np.uint8)
            off = (4 - raw.ctypes.data) % 16
            b._bufs["obs"] = raw[off:off + o2.nbytes].view(np.float32).reshape(o2.shape)
            assert b._bufs["obs"].ctypes.data % 16 == 4


@pytest.mark.parametrize("domain,side,pins", [
    ("maze", 48, ("player", "door")),
    ("dungeon", 40, ("player", "key", "door")),
    ("maze", 16, ("player", "door")),  # lane team of 16 (forced below)
])
def test_lane_team_first_touch_depths(domain, side, pins, monkeypatch):
    """bfs_touch advances two BFS layers per round of team votes and resolves
    the touched layer afterwards (repo:paper_2408_12525_b200/csrc/team.cuh):
    path lengths of both parities, endpoint legs (dungeon) and unreachable
    flags must equal the oracle's (problems.py:176-243) on every step."""
    monkeypatch.setenv("LG_FORCE_TEAM", "1")
    cfg = EnvConfig(domain=domain, max_width=side, max_height=side, obs_size=9, pinpoints=pins)
    n = 128
    env = BatchEnv(cfg, n, seed=3)
    ref = O.OracleBatchEnv(cfg, n, seed=3)
    assert np.array_equal(_np(env.reset()), ref.reset())
    act = np.random.default_rng(5)
    seen = set()
    for t in range(20):
        a = act.integers(0, cfg.n_actions, size=n)
        o2, r2, d2, _ = ref.step(a)
        o1, r1, d1, _ = env.step(a)
        assert np.array_equal(_np(r1), r2), t
        assert np.array_equal(_np(d1), d2), t
        assert np.array_equal(_np(o1), o2), t
        s1, s2 = env.state_dict(), ref.state_dict()
        assert np.array_equal(s1["values"], s2["values"]), t
        assert np.array_equal(s1["unreach"], s2["unreach"]), t
        seen.update(int(v) % 2 for v in s2["values"][0] if v > 0)
    assert seen == {0, 1}  # touched at even and at odd depths


INC_CASES = [
    # (EnvConfig kwargs, envs, steps): lane-team kernels whose steps update the
    # region count incrementally (TeamK::regions_delta)
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 512, 150),    # c4 shape (G64)
    (dict(domain="maze", representation="turtle"), 2048, 300),                     # c2 shape (G16)
    (dict(domain="dungeon", max_width=30, max_height=24, obs_size=9,
          pinpoints=("player", "key", "door")), 600, 200),                         # G32, dungeon open set
    (dict(domain="binary", max_width=40, max_height=40, obs_size=5, randomize_shape=True,
          max_steps=60), 600, 200),                                                # G64, resets mid-run
]


@pytest.mark.parametrize("case", range(len(INC_CASES)))
def test_incremental_region_count_against_oracle(case):
    """Every step's region count (and all other metrics) equals the oracle's
    full recomputation, across auto-resets and after a state import (which
    drops the 'count is exact' bit, so the next write recomputes in full)."""
    kw, n, steps = INC_CASES[case]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=case)
    ref = O.OracleBatchEnv(cfg, n, seed=case)
    assert np.array_equal(_np(env.reset()), ref.reset())
    act = np.random.default_rng(100 + case)
    for t in range(steps):
        a = act.integers(0, cfg.n_actions, size=n)
        _, r1, d1, _ = env.step(a)
        _, r2, d2, _ = ref.step(a)
        assert np.array_equal(_np(r1), r2), t
        if t % 10 == 9:
            s1, s2 = env.state_dict(), ref.state_dict()
            assert np.array_equal(s1["values"], s2["values"]), t
        if t == steps // 2:  # round-trip through a state import mid-run
            twin = BatchEnv(cfg, n, seed=999)
            twin.load_state_dict(env.state_dict())
            env = twin
    s1, s2 = env.state_dict(), ref.state_dict()
    for k in ("tiles", "values", "unreach", "prev_loss", "rng"):
        assert np.array_equal(s1[k], s2[k]), k


def test_envs_on_two_devices_in_one_process():
    """The dynamic shared-memory limit is raised per (kernel, device): envs on
    cuda:0 and cuda:1 in one process both launch kernels needing > 48 KB
    (dungeon narrow obs 31 in solo warp mode: 62 KB per 64-thread block)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cfg = EnvConfig(domain="dungeon")
    n = 20000
    outs = []
    for d in ("cuda:0", "cuda:1"):
        env = BatchEnv(cfg, n, seed=1, device=d)
        env.reset()
        a = np.random.default_rng(0).integers(0, cfg.n_actions, size=n)
        outs.append(_np(env.step(a)[0]))
        assert torch.cuda.current_device() == 0  # the caller's device is restored
    assert np.array_equal(outs[0], outs[1])
