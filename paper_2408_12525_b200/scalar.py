"""Scalar facade: one environment at a time (reference env.py:602-649).

``reset(config, rng)``, ``step(state, action)``, ``observe(state)``,
``next_pos(state)`` and ``rng_from_state`` with the reference's semantics:
states are immutable snapshots (``EnvState``), ``step`` is pure and does not
auto-reset, and the generator handed to ``reset`` is advanced in place. Every
call runs the same CUDA kernels as the batch path on a one-env batch (the
reference's scalar API is likewise its batch code at B=1, env.py:646-649), so
scalar and batched trajectories agree bit for bit.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib
from .config import EnvConfig
from .tiles import Domain


@dataclass(frozen=True)
class Shape:
    width: int
    height: int

    @property
    def area(self) -> int:
        return self.width * self.height


@dataclass(frozen=True, eq=False)
class TileGrid:
    """tiles/active/frozen planes of one level (reference grid.py:48-102)."""

    domain: Domain
    tiles: np.ndarray
    active: np.ndarray
    frozen: np.ndarray

    @property
    def height(self) -> int:
        return int(self.tiles.shape[0])

    @property
    def width(self) -> int:
        return int(self.tiles.shape[1])

    def validate(self) -> None:
        """Structural invariants (reference grid.py:89-102), ValueError on failure."""
        b = self.domain.border_id
        off = ~self.active
        if np.any(self.tiles[off] != b):
            raise ValueError("inactive cell holds a non-border tile")
        if np.any(self.tiles[self.active] == b):
            raise ValueError("active cell holds the border tile")
        if np.any(self.tiles > b):
            raise ValueError("tile id out of range for domain")
        if not np.all(self.frozen[off]):
            raise ValueError("inactive cell is not frozen")

    def __eq__(self, other) -> bool:
        return (isinstance(other, TileGrid) and self.domain.name == other.domain.name
                and np.array_equal(self.tiles, other.tiles)
                and np.array_equal(self.active, other.active)
                and np.array_equal(self.frozen, other.frozen))


@dataclass(frozen=True)
class MetricVector:
    values: dict
    unreachable: frozenset

    def __getitem__(self, name: str) -> int:
        return self.values[name]


@dataclass(frozen=True)
class EnvState:
    """Immutable snapshot of one environment (reference env.py:127-147)."""

    config: EnvConfig
    grid: TileGrid
    shape: Shape
    pos: tuple
    pos_idx: int
    order: np.ndarray
    t: int
    changes: int
    targets: dict
    metrics: MetricVector
    prev_loss: float
    ep_reward: float
    ep_start_loss: float
    max_steps: int
    rng_state: dict
    metric_seed: int | None
    done: bool
    extra: dict = field(default_factory=dict, compare=False, repr=False)


_CACHE: dict[str, Any] = {}


def _env_for(config: EnvConfig):
    from .env import BatchEnv
    key = repr(config)
    env = _CACHE.get(key)
    if env is None:
        env = BatchEnv(config, 1, seed=0)
        _CACHE[key] = env
    return env


def _state_from_row(config: EnvConfig, sd: dict, done: bool) -> EnvState:
    d = config.domain_obj
    names = d.metric_names
    h, w = (int(x) for x in sd["shape_hw"][0])
    n = int(sd["order_len"][0])
    order = sd["order"][0, :n].copy()
    pos_idx = int(sd["pos_idx"][0])
    if config.representation == "turtle":
        pos = (int(sd["pos"][0, 0]), int(sd["pos"][0, 1]))
    else:
        pos = divmod(int(order[pos_idx % n]), config.max_width) if n else (0, 0)
    return EnvState(
        config=config,
        grid=TileGrid(d, sd["tiles"][0].copy(), sd["active"][0].copy(), sd["frozen"][0].copy()),
        shape=Shape(width=w, height=h),
        pos=(int(pos[0]), int(pos[1])),
        pos_idx=pos_idx,
        order=order,
        t=int(sd["t"][0]),
        changes=int(sd["changes"][0]),
        targets={m: (int(sd["lo"][k, 0]), int(sd["hi"][k, 0])) for k, m in enumerate(names)},
        metrics=MetricVector(values={m: int(sd["values"][k, 0]) for k, m in enumerate(names)},
                             unreachable=frozenset(m for k, m in enumerate(names) if sd["unreach"][k, 0])),
        prev_loss=float(sd["prev_loss"][0]),
        ep_reward=float(sd["ep_reward"][0]),
        ep_start_loss=float(sd["ep_start_loss"][0]),
        max_steps=int(sd["max_steps"][0]),
        rng_state=sd["rng_states"][0],
        metric_seed=int(sd["metric_seeds"][0]) if config.deterministic_metrics else None,
        done=done,
        extra={"pos_arr": sd["pos"][0].copy()},
    )


def _row_from_state(st: EnvState) -> dict:
    cfg = st.config
    d = cfg.domain_obj
    names = d.metric_names
    H, W = cfg.max_height, cfg.max_width
    order = np.full((1, H * W), -1, dtype=np.int32)
    order[0, : st.order.size] = st.order
    return {
        "tiles": st.grid.tiles[None].astype(np.uint8), "active": st.grid.active[None],
        "frozen": st.grid.frozen[None],
        "shape_hw": np.array([[st.shape.height, st.shape.width]], dtype=np.int64),
        "order": order, "order_len": np.array([st.order.size], dtype=np.int64),
        "pos_idx": np.array([st.pos_idx], dtype=np.int64),
        "pos": np.array([list(st.pos)], dtype=np.int64),
        "t": np.array([st.t], dtype=np.int64), "changes": np.array([st.changes], dtype=np.int64),
        "max_steps": np.array([st.max_steps], dtype=np.int64),
        "lo": np.array([[st.targets[m][0]] for m in names], dtype=np.int64),
        "hi": np.array([[st.targets[m][1]] for m in names], dtype=np.int64),
        "values": np.array([[st.metrics.values[m]] for m in names], dtype=np.int64),
        "unreach": np.array([[m in st.metrics.unreachable] for m in names], dtype=bool),
        "prev_loss": np.array([st.prev_loss]), "ep_reward": np.array([st.ep_reward]),
        "ep_start_loss": np.array([st.ep_start_loss]),
        "metric_seeds": np.array([st.metric_seed or 0], dtype=np.int64),
        "rng_states": [st.rng_state], "started": np.array([True]),
    }


def rng_from_state(state: dict) -> np.random.Generator:
    """Generator continuing a snapshot's stream (reference env.py:470-475)."""
    bg = np.random.PCG64()
    bg.state = state
    return np.random.Generator(bg)


def spawn_rngs(seed: int, n: int) -> list[np.random.Generator]:
    """Per-row generators of a batch (reference env.py:591-594)."""
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(n)]


def reset(config: EnvConfig, rng: np.random.Generator) -> tuple[EnvState, np.ndarray]:
    """Start one episode drawing from ``rng`` (advanced in place); returns
    (state, first observation) -- reference env.py:602-608."""
    env = _env_for(config)
    H, W, M = config.max_height, config.max_width, len(config.domain_obj.metric_names)
    blank = {
        "tiles": np.zeros((1, H, W), np.uint8), "active": np.zeros((1, H, W), bool),
        "frozen": np.ones((1, H, W), bool), "shape_hw": np.array([[H, W]], np.int64),
        "order": np.full((1, H * W), -1, np.int32), "order_len": np.ones(1, np.int64),
        "pos_idx": np.zeros(1, np.int64), "pos": np.zeros((1, 2), np.int64),
        "t": np.zeros(1, np.int64), "changes": np.zeros(1, np.int64),
        "max_steps": np.ones(1, np.int64), "lo": np.zeros((M, 1), np.int64),
        "hi": np.zeros((M, 1), np.int64), "values": np.zeros((M, 1), np.int64),
        "unreach": np.zeros((M, 1), bool), "prev_loss": np.zeros(1), "ep_reward": np.zeros(1),
        "ep_start_loss": np.zeros(1), "metric_seeds": np.zeros(1, np.int64),
        "rng_states": [rng.bit_generator.state], "started": np.array([False]),
    }
    env.load_state_dict(blank)
    obs = env.reset().cpu().numpy()[0]
    sd = env.state_dict()
    rng.bit_generator.state = sd["rng_states"][0]
    return _state_from_row(config, sd, done=False), obs


def step(state: EnvState, action: int) -> tuple[EnvState, float, bool, dict]:
    """One pure transition without auto-reset (reference env.py:611-630)."""
    if state.done:
        raise ValueError("episode is done; reset first")
    cfg = state.config
    if not 0 <= int(action) < cfg.n_actions:
        raise ValueError("action id out of range")
    env = _env_for(cfg)
    env.load_state_dict(_row_from_state(state))
    t = env._torch
    a = t.tensor([int(action)], dtype=t.int64, device=env.device)
    reward = t.empty(1, dtype=t.float64, device=env.device)
    done = t.empty(1, dtype=t.bool, device=env.device)
    info = env._info_buffers()
    ci = _lib.LgInfo(*[ctypes.c_void_p(info[k].data_ptr()) for k in
                       ("terminal", "episode_reward", "episode_length", "episode_start_loss",
                        "final_loss")])
    with t.cuda.device(env.device):
        _lib.check(_lib.load().lg_step_flags(env.handle, ctypes.c_void_p(a.data_ptr()), None,
                                             ctypes.c_void_p(reward.data_ptr()),
                                             ctypes.c_void_p(done.data_ptr()), ctypes.byref(ci), None,
                                             _lib.STEP_NO_AUTO_RESET,
                                             ctypes.c_void_p(t.cuda.current_stream(env.device).cuda_stream)))
    d = bool(done.item())
    new_state = _state_from_row(cfg, env.state_dict(), done=d)
    out: dict[str, Any] = {"changed": new_state.changes > state.changes, "loss": new_state.prev_loss,
                           "metrics": new_state.metrics}
    if d:
        out.update(episode_reward=float(info["episode_reward"].item()),
                   episode_length=int(info["episode_length"].item()),
                   episode_start_loss=float(info["episode_start_loss"].item()),
                   final_loss=float(info["final_loss"].item()))
    return new_state, float(reward.item()), d, out


def observe(state: EnvState) -> np.ndarray:
    """Observation of a snapshot (reference env.py:633-635)."""
    env = _env_for(state.config)
    env.load_state_dict(_row_from_state(state))
    return env.observe().cpu().numpy()[0]


def next_pos(state: EnvState) -> tuple[int, int]:
    """Scan cell after the current step, wrapping (reference env.py:638-643)."""
    if state.done:
        raise ValueError("episode is done")
    nxt = int(state.order[(state.pos_idx + 1) % state.order.size])
    return divmod(nxt, state.grid.tiles.shape[1])


# ---------------------------------------------------------------------------
# designer edits (reference env.py:657-715): host bookkeeping of the scan
# order, metrics and loss recomputed by the CUDA kernels (lg_recompute)
# ---------------------------------------------------------------------------


def _scan_order(active: np.ndarray, frozen: np.ndarray) -> np.ndarray:
    """Editable cells in boustrophedon order (reference env.py:155-178)."""
    h, w = active.shape
    out = []
    for r in range(h):
        cols = range(w) if r % 2 == 0 else range(w - 1, -1, -1)
        out.extend(r * w + c for c in cols if active[r, c] and not frozen[r, c])
    return np.array(out, dtype=np.int32)


def _serp_rank(h: int, w: int) -> np.ndarray:
    rank = np.empty(h * w, dtype=np.int64)
    k = 0
    for r in range(h):
        for c in (range(w) if r % 2 == 0 else range(w - 1, -1, -1)):
            rank[r * w + c] = k
            k += 1
    return rank


def _device_recompute(state: EnvState, reprice_only: bool) -> EnvState:
    env = _env_for(state.config)
    env.load_state_dict(_row_from_state(state))
    t = env._torch
    with t.cuda.device(env.device):
        _lib.check(_lib.load().lg_recompute(env.handle, None, int(reprice_only),
                                            ctypes.c_void_p(t.cuda.current_stream(env.device).cuda_stream)))
    return _state_from_row(state.config, env.state_dict(), done=state.done)


def _after_grid_edit(state: EnvState, tiles: np.ndarray, frozen: np.ndarray) -> EnvState:
    active = state.grid.active
    order = _scan_order(active, frozen)
    if order.size == 0:
        raise ValueError("edit would leave no editable cells")
    h, w = tiles.shape
    rank = _serp_rank(h, w)
    old_cell = int(state.order[state.pos_idx])
    pos_idx = int(np.searchsorted(rank[order], rank[old_cell])) % order.size  # same cell or next
    flat = int(order[pos_idx])
    edited = EnvState(**{**state.__dict__, "grid": TileGrid(state.grid.domain, tiles, active, frozen),
                         "order": order, "pos_idx": pos_idx, "pos": divmod(flat, w)})
    return _device_recompute(edited, reprice_only=False)


def _pin_checks(state: EnvState, row: int, col: int):
    g = state.grid
    if not (0 <= row < g.tiles.shape[0] and 0 <= col < g.tiles.shape[1]) or not g.active[row, col]:
        raise ValueError(f"cell ({row}, {col}) is not inside the active map")


def with_pin(state: EnvState, row: int, col: int, tile) -> EnvState:
    """Pin a tile mid-episode (reference env.py:657-661, grid.pin_cell)."""
    d = state.config.domain_obj
    tid = d.tile_id(tile) if isinstance(tile, str) else int(tile)
    if d.tile_name(tid) not in d.pivotal:
        raise ValueError(f"tile {d.tile_name(tid)!r} is not pinnable in domain {d.name!r}")
    _pin_checks(state, row, col)
    tiles, frozen = state.grid.tiles.copy(), state.grid.frozen.copy()
    tiles[row, col] = tid
    frozen[row, col] = True
    return _after_grid_edit(state, tiles, frozen)


def without_pin(state: EnvState, row: int, col: int) -> EnvState:
    """Release a pinned cell back into the scan (reference env.py:664-667)."""
    _pin_checks(state, row, col)
    if not state.grid.frozen[row, col]:
        raise ValueError(f"cell ({row}, {col}) is not pinned")
    frozen = state.grid.frozen.copy()
    frozen[row, col] = False
    return _after_grid_edit(state, state.grid.tiles.copy(), frozen)


def with_target(state: EnvState, metric: str, value: int) -> EnvState:
    """Point target for one metric, loss repriced (reference env.py:670-681)."""
    d = state.config.domain_obj
    if metric not in d.metric_names:
        raise ValueError(f"unknown metric {metric!r}")
    cap = state.shape.area
    if not 0 <= value <= cap:
        raise ValueError(f"target {value} outside [0, {cap}]")
    targets = dict(state.targets)
    targets[metric] = (int(value), int(value))
    return _device_recompute(EnvState(**{**state.__dict__, "targets": targets}), reprice_only=True)
