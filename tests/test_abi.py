"""C-ABI library: loads, exports every declared symbol, host-side seeding. CPU only."""
import os
import re

import numpy as np
import pytest

from paper_2408_12525_b200 import _lib
from paper_2408_12525_b200.config import EnvConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pcgrl_b200.h")).read()
    return sorted(set(re.findall(r"\b(lg_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.lg_version().decode().endswith("sm_100a")


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(8|9)\d", out)


def test_host_seed_streams_match_numpy():
    from paper_2408_12525_b200.env import spawn_streams
    for seed in (0, 5, 2 ** 40 + 3):
        got = spawn_streams(seed, 50, offset=1000)
        kids = np.random.SeedSequence(seed).spawn(1050)[1000:]
        for i, k in enumerate(kids):
            st = np.random.default_rng(k).bit_generator.state["state"]
            m = (1 << 64) - 1
            want = [st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m]
            assert [int(x) for x in got[i, :4]] == want


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        EnvConfig(domain="binary", obs_size=2)
    with pytest.raises(ValueError):
        EnvConfig(domain="maze", pinpoints=("wall",))
    with pytest.raises(ValueError):
        EnvConfig(domain="binary", controllable=("path_length",))
    with pytest.raises(ValueError):
        EnvConfig(domain="binary", max_width=2)
    with pytest.raises(ValueError):
        EnvConfig(domain="binary", init_mode="sparse")
    with pytest.raises(KeyError):
        EnvConfig(domain="castle")
    with pytest.raises(ValueError):
        EnvConfig(representation="diagonal")
    EnvConfig(domain="binary", max_width=16, max_height=16, obs_size=31).check_obs_invariant()
    with pytest.raises(ValueError):
        EnvConfig(domain="binary", max_width=8, max_height=8, obs_size=31).check_obs_invariant()
    assert EnvConfig(domain="maze", representation="turtle").n_actions == 8
    assert EnvConfig(domain="dungeon", representation="wide").n_actions == 16 * 16 * 6
    assert EnvConfig(domain="dungeon", representation="wide").observation_shape == (8, 16, 16)
    assert EnvConfig(domain="maze", controllable=("path_length",)).observation_shape == (7, 31, 31)


def test_struct_layouts_match_the_header(tmp_path):
    import ctypes
    import shutil
    import subprocess
    cc = shutil.which("gcc") or "/usr/bin/gcc"
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "pcgrl_b200.h"\n'
                   'int main(){printf("%zu %zu %zu %zu\\n", sizeof(lg_config), sizeof(lg_state),'
                   ' sizeof(lg_desc), sizeof(lg_info));}\n')
    exe = tmp_path / "sz"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.LgConfig), ctypes.sizeof(_lib.LgState),
                   ctypes.sizeof(_lib.LgDesc), ctypes.sizeof(_lib.LgInfo)]
