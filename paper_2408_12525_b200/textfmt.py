"""Text codec and episode traces for device states.

The reference's plain-text grid format (`levelgen/textfmt.py:1-85`) and the
`play` command's frames and JSONL trace records (`levelgen/cli.py:272-362`),
applied to states that live on the GPU: ``BatchEnv.grid_view(i)`` /
``snapshot(i)`` and the scalar facade's ``EnvState`` all hand out a
``TileGrid`` that renders here.

Format: one character per cell (``TILE_CHARS``), one line per row; ``%`` is a
cell outside the active map. If any active cell is frozen, a mask block of
``!``-prefixed lines follows (``*`` frozen, ``.`` free); otherwise frozen is
implied to be exactly the inactive cells and the block is omitted.
"""
from __future__ import annotations

import json
from typing import Callable, Iterable

import numpy as np

from .tiles import Domain

MASK_PREFIX = "!"
MASK_FROZEN = "*"
MASK_FREE = "."


def render_text(grid) -> str:
    """TileGrid -> text (reference textfmt.py:26-37)."""
    d = grid.domain
    chars = np.array([d.char_of(t) for t in range(d.border_id + 1)])
    rows = ["".join(chars[np.asarray(grid.tiles[r], dtype=np.int64)])
            for r in range(grid.tiles.shape[0])]
    frozen = np.asarray(grid.frozen, dtype=bool)
    if (frozen & np.asarray(grid.active, dtype=bool)).any():
        mask = np.where(frozen, MASK_FROZEN, MASK_FREE)
        rows += [MASK_PREFIX + "".join(m) for m in mask]
    return "\n".join(rows) + "\n"


def parse_text(domain: Domain, text: str):
    """text -> TileGrid (reference textfmt.py:40-85); ValueError on ragged rows,
    characters the domain does not have, or a malformed mask block."""
    from .scalar import TileGrid

    lines = [ln for ln in text.splitlines() if ln.strip()]
    body = [ln for ln in lines if not ln.startswith(MASK_PREFIX)]
    masks = [ln[len(MASK_PREFIX):] for ln in lines if ln.startswith(MASK_PREFIX)]
    if not body:
        raise ValueError("empty level text")
    w = len(body[0])
    if w == 0 or any(len(ln) != w for ln in body):
        raise ValueError("ragged level text")
    lut = {}
    tiles = np.empty((len(body), w), dtype=np.uint8)
    for r, ln in enumerate(body):
        for c, ch in enumerate(ln):
            if ch not in lut:
                try:
                    lut[ch] = domain.id_of_char(ch)
                except KeyError as e:
                    raise ValueError(str(e)) from None
            tiles[r, c] = lut[ch]
    active = tiles != domain.border_id
    if masks:
        if len(masks) != len(body) or any(len(m) != w for m in masks):
            raise ValueError("frozen mask does not match level dimensions")
        bad = {ch for m in masks for ch in m} - {MASK_FROZEN, MASK_FREE}
        if bad:
            raise ValueError(f"bad mask character {sorted(bad)[0]!r}")
        frozen = np.array([[ch == MASK_FROZEN for ch in m] for m in masks], dtype=bool)
        if (~frozen & ~active).any():
            raise ValueError("inactive cells must be frozen")
    else:
        frozen = ~active
    grid = TileGrid(domain=domain, tiles=tiles, active=active, frozen=frozen)
    grid.validate()
    return grid


def frame(state) -> str:
    """A play frame: the grid text with ``@`` at the agent cell (cli.py:272-281)."""
    lines = render_text(state.grid).splitlines()
    r, c = state.pos
    lines[r] = lines[r][:c] + "@" + lines[r][c + 1:]
    return "\n".join(lines)


def trace_record(state, action: int, reward: float) -> dict:
    """One JSONL trace row of ``levelgen play --trace`` (cli.py:348-356)."""
    return {
        "step": int(state.t),
        "action": int(action),
        "reward": float(reward),
        "loss": float(state.prev_loss),
        "metrics": {k: int(v) for k, v in state.metrics.values.items()},
        "pos": [int(p) for p in state.pos],
    }


def play(config, seed: int, policy: Callable[[np.ndarray], int] | None = None,
         trace: Iterable | None = None) -> list[str]:
    """One episode on the GPU scalar facade, the same text ``levelgen play``
    prints (cli.py:318-362): reset from ``default_rng(seed)``, random actions
    from ``default_rng(seed + 1)`` unless ``policy(obs) -> action`` is given.
    Returns the printed lines; trace rows are appended to ``trace`` (a list)
    or written as JSON lines (a writable file)."""
    from . import scalar

    rng = np.random.default_rng(seed)
    action_rng = np.random.default_rng(seed + 1)
    state, obs = scalar.reset(config, rng)
    out = [f"step 0  loss {state.prev_loss:g}", frame(state)]
    while not state.done:
        if policy is None:
            action = int(action_rng.integers(config.n_actions))
        else:
            action = int(policy(obs))
        state, reward, _, _ = scalar.step(state, action)
        obs = scalar.observe(state)
        out.append(f"step {state.t}  action {action}  reward {reward:g}  loss {state.prev_loss:g}")
        out.append(frame(state))
        if trace is not None:
            row = trace_record(state, action, reward)
            if hasattr(trace, "write"):
                trace.write(json.dumps(row) + "\n")
            else:
                trace.append(row)
    out.append(f"episode reward {state.ep_reward:g}  "
               f"start loss {state.ep_start_loss:g}  final loss {state.prev_loss:g}")
    return out
