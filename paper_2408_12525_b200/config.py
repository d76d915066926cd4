"""``EnvConfig``: the static description of one environment family.

Field-compatible with the reference (`levelgen/env.py:42-124`), plus
``representation`` ("narrow" | "turtle" | "wide", default "narrow"); the
turtle and wide action spaces are defined in DESIGN.md ("Representations")
because the reference declares them a non-goal.
Validation raises the same exception types as the reference.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .tiles import Domain, get_domain

MIN_SIDE = 3
REPRESENTATIONS = ("narrow", "turtle", "wide")
# Kernel limits (csrc/env_kernels.cuh): one row of the max grid is one
# 64-bit word and one env's rows fit a 32-lane team with two rows per lane.
MAX_SIDE_DEVICE = 64
MAX_WINDOW_DEVICE = 128


@dataclass(frozen=True)
class EnvConfig:
    domain: str = "binary"
    max_width: int = 16
    max_height: int = 16
    obs_size: int = 31
    randomize_shape: bool = False
    pinpoints: tuple[str, ...] = ()
    controllable: tuple[str, ...] = ()
    init_mode: str | None = None
    init_weights: dict[str, float] | None = None
    max_steps: int | None = None
    change_budget: int | None = None
    loss_weights: dict[str, float] = field(default_factory=dict)
    deterministic_metrics: bool = False
    representation: str = "narrow"

    def __post_init__(self) -> None:
        d = get_domain(self.domain)  # KeyError for unknown domains
        if self.max_width < MIN_SIDE or self.max_height < MIN_SIDE:
            raise ValueError(f"max shape below {MIN_SIDE}x{MIN_SIDE}")
        if self.obs_size < 3:
            raise ValueError("obs_size must be at least 3")
        if self.init_mode not in (None, "weighted", "empty"):
            raise ValueError(f"unknown init_mode {self.init_mode!r}")
        bad = [t for t in self.pinpoints if t not in d.pivotal]
        if bad:
            raise ValueError(f"tile {bad[0]!r} is not pinnable in domain {d.name!r}")
        unknown = set(self.controllable) - set(d.metric_names)
        if unknown:
            raise ValueError(f"unknown controllable metrics {sorted(unknown)}")
        unknown = set(self.loss_weights) - set(d.metric_names)
        if unknown:
            raise ValueError(f"unknown loss weight keys {sorted(unknown)}")
        if self.max_steps is not None and self.max_steps < 1:
            raise ValueError("max_steps must be positive")
        if self.change_budget is not None and self.change_budget < 1:
            raise ValueError("change_budget must be positive")
        if self.representation not in REPRESENTATIONS:
            raise ValueError(f"unknown representation {self.representation!r}")

    @property
    def domain_obj(self) -> Domain:
        return get_domain(self.domain)

    @property
    def n_actions(self) -> int:
        n = self.domain_obj.n_tiles
        if self.representation == "turtle":
            return 4 + n
        if self.representation == "wide":
            return self.max_width * self.max_height * n
        return n + 1

    def weights(self) -> dict[str, float]:
        w = {m: 1.0 for m in self.domain_obj.metric_names}
        w.update(self.loss_weights)
        return w

    def check_obs_invariant(self) -> None:
        limit = 2 * max(self.max_width, self.max_height) - 1
        if self.obs_size > limit:
            raise ValueError(f"obs_size {self.obs_size} exceeds 2*max(width,height)-1 = {limit}")

    def control_order(self) -> tuple[str, ...]:
        return tuple(m for m in self.domain_obj.metric_names if m in self.controllable)

    def observation_channels(self) -> int:
        return self.domain_obj.n_tiles + 2 + len(self.control_order())

    @property
    def observation_shape(self) -> tuple[int, int, int]:
        c = self.observation_channels()
        if self.representation == "wide":
            return (c, self.max_height, self.max_width)
        return (c, self.obs_size, self.obs_size)

    def init_cdf(self) -> np.ndarray:
        """numpy ``Generator.choice`` cdf of the init weights (grid.py:153-191)."""
        d = self.domain_obj
        cdf = normalize_weights(d, self.init_weights if self.init_weights else d.default_init_weights).cumsum()
        cdf /= cdf[-1]
        return cdf


def normalize_weights(domain: Domain, weights) -> np.ndarray:
    """grid.normalize_weights (grid.py:153-166): weights keyed by tile name or
    id -> dense probability vector, with the reference's errors."""
    vec = np.zeros(domain.n_tiles, dtype=np.float64)
    for key, w in weights.items():
        tid = domain.tile_id(key) if isinstance(key, str) else int(key)
        if not 0 <= tid < domain.n_tiles:
            raise ValueError(f"weight for non-writable tile id {tid}")
        if w < 0:
            raise ValueError(f"negative weight for tile {key!r}")
        vec[tid] = w
    total = float(vec.sum())
    if total <= 0:
        raise ValueError("tile weights sum to zero")
    return vec / total
