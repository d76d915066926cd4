"""Text codec + play traces against the live reference's output
(tests/golden/make_textfmt_golden.py). The codec tests are CPU-only; the play
and device-grid tests run the GPU scalar facade."""
import io
import json
import os

import numpy as np
import pytest

from paper_2408_12525_b200 import get_domain
from paper_2408_12525_b200.config import EnvConfig
from paper_2408_12525_b200.scalar import TileGrid
from paper_2408_12525_b200.textfmt import parse_text, render_text

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "textfmt.json")))


def _grid(g):
    return TileGrid(domain=get_domain(g["domain"]), tiles=np.array(g["tiles"], dtype=np.uint8),
                    active=np.array(g["active"], dtype=bool), frozen=np.array(g["frozen"], dtype=bool))


@pytest.mark.parametrize("k", range(len(GOLD["grids"])))
def test_render_and_parse_match_reference(k):
    g = GOLD["grids"][k]
    grid = _grid(g)
    assert render_text(grid) == g["text"]
    assert parse_text(grid.domain, g["text"]) == grid


def test_round_trip_plain_and_masked():
    # reference tests/test_grid.py:149-162
    g = parse_text(get_domain("binary"), "..#\n#..\n")
    assert render_text(g) == "..#\n#..\n"
    assert (g.frozen == ~g.active).all()
    maze = get_domain("maze")
    g = parse_text(maze, "P.#%\n.D.%\n%%%%\n!*..*\n!.*.*\n!****\n")
    assert g.active[:2, :3].all() and not g.active[2].any()
    assert g.frozen[0, 0] and g.frozen[1, 1] and not g.frozen[0, 1]
    assert parse_text(maze, render_text(g)) == g


@pytest.mark.parametrize("text", [
    "..\n.\n",              # ragged
    "..P\n...\n",           # tile the domain does not have
    "",                     # empty
    "..\n..\n!..\n",        # mask rows incomplete
    ".%\n..\n!.x\n!..\n",   # bad mask character
    ".%\n..\n!..\n!..\n",   # inactive cell left unfrozen
])
def test_parse_errors(text):
    # reference tests/test_grid.py:165-177
    with pytest.raises(ValueError):
        parse_text(get_domain("binary"), text)


def _cfg(kw):
    kw = dict(kw)
    if "pinpoints" in kw:
        kw["pinpoints"] = tuple(kw["pinpoints"])
    return EnvConfig(**kw)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(GOLD["plays"])))
def test_play_matches_reference_cli(k):
    from paper_2408_12525_b200.textfmt import play
    p = GOLD["plays"][k]
    rows = []
    lines = play(_cfg(p["config"]), p["seed"], trace=rows)
    assert "\n".join(lines) + "\n" == p["stdout"]
    assert rows == p["trace"]
    buf = io.StringIO()
    play(_cfg(p["config"]), p["seed"], trace=buf)
    assert [json.loads(ln) for ln in buf.getvalue().splitlines()] == p["trace"]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(GOLD["grids"])))
def test_device_grid_renders_like_reference(k):
    # the make_textfmt_golden.py GRIDS episodes, run on the GPU scalar facade
    from paper_2408_12525_b200 import scalar
    g = GOLD["grids"][k]
    cfg, seed = _cfg(g["config"]), g["seed"]
    st, _ = scalar.reset(cfg, np.random.default_rng(seed))
    for _ in range(5):
        st, *_ = scalar.step(st, int(np.random.default_rng(seed + 7).integers(cfg.n_actions)))
    assert render_text(st.grid) == GOLD["grids"][k]["text"]
