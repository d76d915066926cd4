"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

The oracle is a scalar C restatement of the reference env step
(`/root/reference/pkg/src/levelgen/env.py:241-467`, `problems.py:105-279`,
`pathfind.py:45-203`, `grid.py:116-225`) and of the numpy random streams it
consumes. It is the parity checker for the CUDA product path and the CPU
baseline timed by ``bench.py``; the product package never imports it.

Parity pinning: ``tests/test_oracle_golden.py`` compares it with fixtures
generated from the live reference (``tests/golden/make_golden.py``) and with
the SURVEY.md Appendix C digests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblgoracle.so")


# Domain tables restated from tiles.py:126-171 (ids are tuple positions).
@dataclass(frozen=True)
class ODomain:
    name: str
    code: int
    tiles: tuple
    pivotal: tuple
    metric_names: tuple
    default_init_mode: str
    default_init_weights: dict

    @property
    def n_tiles(self) -> int:
        return len(self.tiles)

    def tile_id(self, name: str) -> int:
        if name == "border":
            return len(self.tiles)
        return self.tiles.index(name)


ODOMAINS = {
    "binary": ODomain("binary", 0, ("air", "wall"), (), ("diameter", "regions"),
                      "weighted", {"air": 0.5, "wall": 0.5}),
    "maze": ODomain("maze", 1, ("air", "wall", "player", "door"), ("player", "door"),
                    ("path_length", "regions", "n_player", "n_door"), "empty",
                    {t: 0.25 for t in ("air", "wall", "player", "door")}),
    "dungeon": ODomain("dungeon", 2, ("air", "wall", "enemy", "key", "door", "player"),
                       ("player", "key", "door"),
                       ("pkd_path", "regions", "n_player", "n_key", "n_door", "n_enemy",
                        "nearest_enemy"), "empty",
                       {t: 1.0 / 6 for t in ("air", "wall", "enemy", "key", "door", "player")}),
}
REPS = {"narrow": 0, "turtle": 1, "wide": 2}


class OrCfg(ctypes.Structure):
    _fields_ = [
        ("domain", ctypes.c_int32), ("representation", ctypes.c_int32),
        ("max_h", ctypes.c_int32), ("max_w", ctypes.c_int32),
        ("obs_size", ctypes.c_int32), ("randomize_shape", ctypes.c_int32),
        ("init_weighted", ctypes.c_int32), ("n_pins", ctypes.c_int32),
        ("pins", ctypes.c_int32 * 16), ("n_ctrl", ctypes.c_int32),
        ("ctrl", ctypes.c_int32 * 8), ("max_steps", ctypes.c_int64),
        ("change_budget", ctypes.c_int64), ("det_metrics", ctypes.c_int32),
        ("_pad", ctypes.c_int32), ("init_cdf", ctypes.c_double * 8),
        ("weights", ctypes.c_double * 8),
    ]


_P = ctypes.c_void_p


class OrState(ctypes.Structure):
    _fields_ = [(n, _P) for n in (
        "tiles", "active", "frozen", "shape_hw", "order", "order_len", "pos_idx", "pos",
        "t", "changes", "max_steps", "lo", "hi", "values", "unreach", "prev_loss",
        "ep_reward", "ep_start_loss", "metric_seeds", "rng")]


_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE, "liblgoracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_last_error.restype = ctypes.c_char_p
        L.or_seed_streams.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _P]
        L.or_seed_plain.argtypes = [ctypes.c_uint64, _P]
        L.or_reset.argtypes = [ctypes.POINTER(OrCfg), ctypes.POINTER(OrState), ctypes.c_int64, _P]
        L.or_step.argtypes = [ctypes.POINTER(OrCfg), ctypes.POINTER(OrState), ctypes.c_int64, _P,
                              _P, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.or_observe.argtypes = [ctypes.POINTER(OrCfg), ctypes.POINTER(OrState), ctypes.c_int64, _P]
        L.or_metrics.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _P, _P,
                                 _P, _P, _P]
        L.or_rng_draw.argtypes = [_P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_int64, _P]
        L.or_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int) -> None:
    if rc != 0:
        raise ValueError(lib().or_last_error().decode())


def _get(cfg, name, default):
    return getattr(cfg, name, default)


def make_cfg(cfg) -> OrCfg:
    """EnvConfig-like object (duck-typed, reference env.py:42-124 fields plus
    ``representation``) -> C struct."""
    d = ODOMAINS[cfg.domain]
    c = OrCfg()
    c.domain = d.code
    c.representation = REPS[_get(cfg, "representation", "narrow")]
    c.max_h, c.max_w = int(cfg.max_height), int(cfg.max_width)
    c.obs_size = int(cfg.obs_size)
    c.randomize_shape = int(bool(cfg.randomize_shape))
    mode = cfg.init_mode or d.default_init_mode
    c.init_weighted = int(mode == "weighted")
    # normalize_weights (grid.py:153-166) then numpy choice cdf
    wts = cfg.init_weights if cfg.init_weights else d.default_init_weights
    vec = np.zeros(d.n_tiles, dtype=np.float64)
    for k, w in wts.items():
        vec[d.tile_id(k) if isinstance(k, str) else int(k)] = w
    p = vec / float(vec.sum())
    cdf = p.cumsum()
    cdf /= cdf[-1]
    for i, v in enumerate(cdf):
        c.init_cdf[i] = float(v)
    pins = [d.tile_id(t) if isinstance(t, str) else int(t) for t in cfg.pinpoints]
    if len(pins) > 16:
        raise ValueError("oracle supports at most 16 pinpoints")
    c.n_pins = len(pins)
    for i, t in enumerate(pins):
        c.pins[i] = t
    ctrl = [i for i, m in enumerate(d.metric_names) if m in cfg.controllable]
    c.n_ctrl = len(ctrl)
    for i, m in enumerate(ctrl):
        c.ctrl[i] = m
    c.max_steps = int(cfg.max_steps) if cfg.max_steps is not None else 0
    c.change_budget = int(cfg.change_budget) if cfg.change_budget is not None else 0
    c.det_metrics = int(bool(cfg.deterministic_metrics))
    lw = dict(cfg.loss_weights or {})
    for i, m in enumerate(d.metric_names):
        c.weights[i] = float(lw.get(m, 1.0))
    return c


def n_actions(cfg) -> int:
    d = ODOMAINS[cfg.domain]
    rep = _get(cfg, "representation", "narrow")
    if rep == "turtle":
        return 4 + d.n_tiles
    if rep == "wide":
        return int(cfg.max_height) * int(cfg.max_width) * d.n_tiles
    return d.n_tiles + 1


def obs_shape(cfg) -> tuple[int, int, int]:
    d = ODOMAINS[cfg.domain]
    c = d.n_tiles + 2 + sum(1 for m in d.metric_names if m in cfg.controllable)
    if _get(cfg, "representation", "narrow") == "wide":
        return (c, int(cfg.max_height), int(cfg.max_width))
    return (c, int(cfg.obs_size), int(cfg.obs_size))


def seed_streams(seed: int, offset: int, n: int) -> np.ndarray:
    out = np.zeros((n, 6), dtype=np.uint64)
    lib().or_seed_streams(int(seed), int(offset), int(n), _ptr(out))
    return out


def seed_plain(seed: int) -> np.ndarray:
    out = np.zeros(6, dtype=np.uint64)
    lib().or_seed_plain(int(seed), _ptr(out))
    return out


def rng_to_numpy_state(row: np.ndarray) -> dict:
    """[6] uint64 -> numpy PCG64 ``bit_generator.state`` dict."""
    s = (int(row[0]) << 64) | int(row[1])
    inc = (int(row[2]) << 64) | int(row[3])
    return {"bit_generator": "PCG64", "state": {"state": s, "inc": inc},
            "has_uint32": int(row[4]), "uinteger": int(row[5])}


def rng_from_numpy_state(st: dict) -> np.ndarray:
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]),
                     int(st["uinteger"])], dtype=np.uint64)


def rng_draw(rng_row: np.ndarray, kind: int, n: int, arg: int = 0, arg2: int = 0) -> np.ndarray:
    out = np.zeros(n * max(1, arg2 if kind == 4 else 1), dtype=np.uint64)
    _check(lib().or_rng_draw(_ptr(rng_row), kind, arg, arg2, n, _ptr(out)))
    return out


def metrics(domain: str, tiles: np.ndarray, active: np.ndarray, rng: np.ndarray | None = None):
    """compute_metrics_batch restated: returns (values [M,B] int64, unreach [M,B] bool);
    ``rng`` ([B,6] uint64) is advanced in place for binary."""
    d = ODOMAINS[domain]
    tiles = np.ascontiguousarray(tiles, dtype=np.uint8)
    active = np.ascontiguousarray(active, dtype=np.uint8)
    b, h, w = tiles.shape
    M = len(d.metric_names)
    vals = np.zeros((M, b), dtype=np.int64)
    unr = np.zeros((M, b), dtype=np.uint8)
    if rng is None:
        rng = np.zeros((b, 6), dtype=np.uint64)
        if domain == "binary":
            raise ValueError("binary metrics need generators")
    _check(lib().or_metrics(d.code, h, w, b, _ptr(tiles), _ptr(active), _ptr(rng), _ptr(vals),
                            _ptr(unr)))
    return vals, unr.astype(bool)


class OracleBatchEnv:
    """The reference ``BatchEnv`` (env.py:486-588) restated over the C oracle.

    ``offset`` selects global env indices ``offset..offset+n-1`` of the
    spawned streams, which is how shards of a multi-GPU batch are checked.
    """

    def __init__(self, config, n_envs: int, seed: int = 0, offset: int = 0):
        self.config = config
        self.cfg = make_cfg(config)
        d = ODOMAINS[config.domain]
        self.domain = d
        B, H, W, M = int(n_envs), int(config.max_height), int(config.max_width), len(d.metric_names)
        self.n_envs = B
        self.n_actions = n_actions(config)
        self.observation_shape = obs_shape(config)
        self.arrays = {
            "tiles": np.full((B, H, W), d.n_tiles, dtype=np.uint8),
            "active": np.zeros((B, H, W), dtype=np.uint8),
            "frozen": np.ones((B, H, W), dtype=np.uint8),
            "shape_hw": np.zeros((B, 2), dtype=np.int64),
            "order": np.full((B, H * W), -1, dtype=np.int32),
            "order_len": np.zeros(B, dtype=np.int64),
            "pos_idx": np.zeros(B, dtype=np.int64),
            "pos": np.zeros((B, 2), dtype=np.int64),
            "t": np.zeros(B, dtype=np.int64),
            "changes": np.zeros(B, dtype=np.int64),
            "max_steps": np.zeros(B, dtype=np.int64),
            "lo": np.zeros((M, B), dtype=np.int64),
            "hi": np.zeros((M, B), dtype=np.int64),
            "values": np.zeros((M, B), dtype=np.int64),
            "unreach": np.zeros((M, B), dtype=np.uint8),
            "prev_loss": np.zeros(B, dtype=np.float64),
            "ep_reward": np.zeros(B, dtype=np.float64),
            "ep_start_loss": np.zeros(B, dtype=np.float64),
            "metric_seeds": np.zeros(B, dtype=np.int64),
            "rng": seed_streams(seed, offset, B),
        }
        self.st = OrState(**{k: _ptr(v) for k, v in self.arrays.items()})
        self._started = False

    def reset(self) -> np.ndarray:
        _check(lib().or_reset(ctypes.byref(self.cfg), ctypes.byref(self.st), self.n_envs, None))
        self._started = True
        return self.observe()

    def step(self, actions):
        if not self._started:
            raise RuntimeError("reset() the batch before stepping")
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.int64))
        if a.shape != (self.n_envs,):
            raise ValueError(f"expected {self.n_envs} actions, got shape {a.shape}")
        B = self.n_envs
        reward = np.zeros(B, dtype=np.float64)
        done = np.zeros(B, dtype=np.uint8)
        term = np.zeros(B, dtype=np.uint8)
        er = np.zeros(B, dtype=np.float64)
        el = np.zeros(B, dtype=np.int64)
        es = np.zeros(B, dtype=np.float64)
        fl = np.zeros(B, dtype=np.float64)
        _check(lib().or_step(ctypes.byref(self.cfg), ctypes.byref(self.st), B, _ptr(a), _ptr(reward),
                             _ptr(done), _ptr(term), _ptr(er), _ptr(el), _ptr(es), _ptr(fl), 1))
        info = {"terminal": term.astype(bool), "episode_reward": er, "episode_length": el,
                "episode_start_loss": es, "final_loss": fl}
        return self.observe(), reward, done.astype(bool), info

    def step_no_obs(self, actions):
        """step() without building the observation (bench sampling helper)."""
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.int64))
        B = self.n_envs
        bufs = [np.zeros(B, dtype=t) for t in (np.float64, np.uint8, np.uint8, np.float64,
                                                np.int64, np.float64, np.float64)]
        _check(lib().or_step(ctypes.byref(self.cfg), ctypes.byref(self.st), B, _ptr(a),
                             *[_ptr(x) for x in bufs], 1))
        return bufs

    def step_no_obs_info(self, actions):
        """step() without the observation: (reward, done, info) (parity helper)."""
        rw, dn, tm, er, el, es, fl = self.step_no_obs(actions)
        info = {"terminal": tm.astype(bool), "episode_reward": er, "episode_length": el,
                "episode_start_loss": es, "final_loss": fl}
        return rw, dn.astype(bool), info

    def observe(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.n_envs,) + self.observation_shape, dtype=np.float32)
        _check(lib().or_observe(ctypes.byref(self.cfg), ctypes.byref(self.st), self.n_envs, _ptr(out)))
        return out

    def state_dict(self) -> dict:
        a = self.arrays
        out = {k: v.copy() for k, v in a.items() if k not in ("rng",)}
        out["active"] = out["active"].astype(bool)
        out["frozen"] = out["frozen"].astype(bool)
        out["unreach"] = out["unreach"].astype(bool)
        out["rng_states"] = [rng_to_numpy_state(r) for r in a["rng"]]
        out["rng"] = a["rng"].copy()
        return out
