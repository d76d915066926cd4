"""Golden fixtures for the text codec and play traces, from the LIVE reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_textfmt_golden.py

Writes ``textfmt.json``: (1) ``render_text`` of grids the reference's own
episodes produce (all three domains, random shapes, pinned cells), with the
planes, so the codec is checked both ways; (2) the stdout and JSONL trace of
``levelgen play random`` (cli.py:318-362) for a few configs, so the GPU
scalar facade's ``textfmt.play`` can be compared line for line.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from click.testing import CliRunner  # noqa: E402
from levelgen import env as E  # noqa: E402
from levelgen.cli import main  # noqa: E402
from levelgen.textfmt import render_text  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (EnvConfig kwargs, --set overrides for `play`, seed)
PLAYS = [
    (dict(max_width=4, max_height=4, obs_size=5, max_steps=6),
     ["env.max_width=4", "env.max_height=4", "env.obs_size=5", "env.max_steps=6"], 0),
    (dict(domain="maze", max_width=4, max_height=4, obs_size=5, max_steps=2, pinpoints=("player", "door")),
     ["env.domain=maze", "env.max_width=4", "env.max_height=4", "env.obs_size=5", "env.max_steps=2",
      "env.pinpoints=[player,door]"], 0),
    (dict(domain="dungeon", max_width=7, max_height=6, obs_size=9, randomize_shape=True,
          pinpoints=("player", "key", "door")),
     ["env.domain=dungeon", "env.max_width=7", "env.max_height=6", "env.obs_size=9",
      "env.randomize_shape=true", "env.pinpoints=[player,key,door]"], 5),
    (dict(domain="binary", max_width=8, max_height=8, obs_size=7, max_steps=40),
     ["env.max_width=8", "env.max_height=8", "env.obs_size=7", "env.max_steps=40"], 3),
]

GRIDS = [
    (dict(domain="binary", max_width=9, max_height=7, randomize_shape=True), 11),
    (dict(domain="maze", max_width=6, max_height=5, pinpoints=("player", "door")), 2),
    (dict(domain="dungeon", max_width=8, max_height=8, randomize_shape=True,
          pinpoints=("player", "key", "door")), 4),
    (dict(domain="dungeon", max_width=5, max_height=9, init_mode="weighted"), 9),
]


def main_() -> None:
    out = {"plays": [], "grids": []}
    runner = CliRunner()
    for kw, sets, seed in PLAYS:
        with tempfile.TemporaryDirectory() as td:
            trace = os.path.join(td, "t.jsonl")
            args = ["play", "random", "--seed", str(seed), "--trace", trace]
            for s in sets:
                args += ["--set", s]
            res = runner.invoke(main, args)
            assert res.exit_code == 0, res.output
            rows = [json.loads(ln) for ln in open(trace).read().splitlines()]
        out["plays"].append({"config": kw, "seed": seed, "stdout": res.output, "trace": rows})
    for kw, seed in GRIDS:
        cfg = E.EnvConfig(**kw)
        st, _ = E.reset(cfg, np.random.default_rng(seed))
        for _ in range(5):
            st, *_ = E.step(st, int(np.random.default_rng(seed + 7).integers(cfg.n_actions)))
        g = st.grid
        out["grids"].append({"config": kw, "seed": seed, "domain": kw["domain"], "text": render_text(g),
                             "tiles": g.tiles.tolist(), "active": g.active.astype(int).tolist(),
                             "frozen": g.frozen.astype(int).tolist()})
    with open(os.path.join(OUT, "textfmt.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote textfmt.json", len(out["plays"]), "plays", len(out["grids"]), "grids")


if __name__ == "__main__":
    main_()
