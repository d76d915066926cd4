"""Tile vocabularies of the three PCGRL problems.

Mirrors the reference domain tables (`levelgen/tiles.py:32-180`): dense tile
ids in declaration order, ``border_id == n_tiles`` for out-of-map cells, the
pinnable ("pivotal") tiles, the passable sets used by the path and region
metrics, and the canonical metric order that fixes the loss accumulation
order. These tables are compiled into the CUDA kernels as template
constants (``Dom<DOM>`` in ``csrc/env_kernels.cuh``); this module is the host-side view.
"""
from __future__ import annotations

from dataclasses import dataclass, field

BORDER = "border"

# printable character per tile name (reference tiles.py:20-29): text codec,
# play frames and traces
TILE_CHARS = {"air": ".", "wall": "#", "player": "P", "door": "D", "key": "K", "enemy": "E",
              BORDER: "%"}


@dataclass(frozen=True)
class Domain:
    name: str
    code: int                       # kernel template id (Dom<code> in csrc/env_kernels.cuh)
    tiles: tuple[str, ...]
    pivotal: tuple[str, ...]
    path_passable: tuple[str, ...]
    region_passable: tuple[str, ...]
    metric_names: tuple[str, ...]
    path_metrics: tuple[str, ...]
    maximize: tuple[str, ...]
    default_init_mode: str
    default_init_weights: dict = field(repr=False, default_factory=dict)

    @property
    def n_tiles(self) -> int:
        return len(self.tiles)

    @property
    def border_id(self) -> int:
        return len(self.tiles)

    @property
    def n_channels_tiles(self) -> int:
        return len(self.tiles) + 1

    def tile_id(self, name: str) -> int:
        if name == BORDER:
            return self.border_id
        if name not in self.tiles:
            raise KeyError(f"domain {self.name!r} has no tile {name!r}")
        return self.tiles.index(name)

    def tile_name(self, tid: int) -> str:
        if tid == self.border_id:
            return BORDER
        if 0 <= tid < len(self.tiles):
            return self.tiles[tid]
        raise KeyError(f"domain {self.name!r} has no tile id {tid}")

    def char_of(self, tid: int) -> str:
        return TILE_CHARS[self.tile_name(tid)]

    def id_of_char(self, ch: str) -> int:
        names = [n for n, c in TILE_CHARS.items() if c == ch and (n == BORDER or n in self.tiles)]
        if not names:
            raise KeyError(f"domain {self.name!r} has no tile for character {ch!r}")
        return self.tile_id(names[0])

    @property
    def pivotal_ids(self) -> tuple[int, ...]:
        return tuple(self.tile_id(t) for t in self.pivotal)


def _even(names):
    return {n: 1.0 / len(names) for n in names}


BINARY = Domain(
    "binary", 0, ("air", "wall"), (), ("air",), ("air",), ("diameter", "regions"), (),
    ("diameter",), "weighted", {"air": 0.5, "wall": 0.5})
MAZE = Domain(
    "maze", 1, ("air", "wall", "player", "door"), ("player", "door"),
    ("air", "player", "door"), ("air", "player", "door"),
    ("path_length", "regions", "n_player", "n_door"), ("path_length",), ("path_length",),
    "empty", _even(("air", "wall", "player", "door")))
DUNGEON = Domain(
    "dungeon", 2, ("air", "wall", "enemy", "key", "door", "player"), ("player", "key", "door"),
    ("air", "player"), ("air", "player", "key", "door"),
    ("pkd_path", "regions", "n_player", "n_key", "n_door", "n_enemy", "nearest_enemy"),
    ("pkd_path", "nearest_enemy"), ("pkd_path",), "empty",
    _even(("air", "wall", "enemy", "key", "door", "player")))

DOMAINS = {d.name: d for d in (BINARY, MAZE, DUNGEON)}


def get_domain(name: str) -> Domain:
    if name not in DOMAINS:
        raise KeyError(f"unknown domain {name!r}; expected one of {sorted(DOMAINS)}")
    return DOMAINS[name]
