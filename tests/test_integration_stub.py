"""the reference-side binding (``levelgen/b200.py``),
run as written from ``integration/levelgen_b200.py``.

The stub imports ``EnvConfig`` from ``levelgen.env`` and ``normalize_weights``
from ``levelgen.grid``. The reference cannot travel to the GPU box, so the
tests mount it under a ``levelgen`` package backed by the field-compatible
mirror (``paper_2408_12525_b200.config``: same fields, ``domain_obj``,
``weights()``, ``observation_channels()``, ``n_actions``, and
``normalize_weights`` = grid.py:153-166). When the reference is importable
(the build container), its own ``EnvConfig`` is checked too.
"""
import importlib.util
import os
import sys
import types

import numpy as np
import pytest

from paper_2408_12525_b200 import _lib
from paper_2408_12525_b200 import config as C
from paper_2408_12525_b200.env import make_lg_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STUB = os.path.join(ROOT, "integration", "levelgen_b200.py")

CONFIGS = [
    dict(domain="binary"),
    dict(domain="maze", pinpoints=("player", "door"), controllable=("path_length", "regions"),
         loss_weights={"regions": 2.0}, max_steps=50),
    dict(domain="dungeon", max_width=12, max_height=9, obs_size=9, randomize_shape=True,
         init_mode="weighted", init_weights={"air": 3.0, "wall": 1.0, "enemy": 0.5}, change_budget=7,
         deterministic_metrics=True),
]


def load_stub(env_mod, grid_mod):
    """Import the stub as levelgen.b200 over the given levelgen.env / .grid."""
    pkg = types.ModuleType("levelgen")
    pkg.__path__ = []
    saved = {k: sys.modules.get(k) for k in ("levelgen", "levelgen.env", "levelgen.grid", "levelgen.b200")}
    sys.modules.update({"levelgen": pkg, "levelgen.env": env_mod, "levelgen.grid": grid_mod})
    os.environ["LEVELGEN_B200_LIB"] = _lib.LIB_PATH
    try:
        spec = importlib.util.spec_from_file_location("levelgen.b200", STUB)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v


def mirror_stub():
    env_mod = types.ModuleType("levelgen.env")
    env_mod.EnvConfig = C.EnvConfig
    grid_mod = types.ModuleType("levelgen.grid")
    grid_mod.normalize_weights = C.normalize_weights
    return load_stub(env_mod, grid_mod)


def _fields(s):
    out = {}
    for name, _ in s._fields_:
        v = getattr(s, name)
        out[name] = list(v) if hasattr(v, "__len__") else v
    return out


@pytest.mark.parametrize("kw", CONFIGS)
def test_stub_config_marshalling_matches_the_mirror(kw):
    stub = mirror_stub()
    cfg = C.EnvConfig(**kw)
    assert _fields(stub._cfg(cfg)) == _fields(make_lg_config(cfg))
    # the stub's struct is the header's lg_config, field for field
    assert [n for n, _ in stub._Cfg._fields_] == [n for n, _ in _lib.LgConfig._fields_]


@pytest.mark.parametrize("kw", CONFIGS)
def test_stub_against_the_reference_envconfig(kw):
    """In the build container: the stub over the reference's own modules."""
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, ref)
    try:
        from levelgen import env as E
        from levelgen import grid as Gr
        stub = load_stub(E, Gr)
        rkw = dict(kw)
        cfg = E.EnvConfig(**rkw)
        assert _fields(stub._cfg(cfg)) == _fields(make_lg_config(C.EnvConfig(**kw)))
    finally:
        sys.path.remove(ref)
        for k in [k for k in sys.modules if k == "levelgen" or k.startswith("levelgen.")]:
            sys.modules.pop(k)


@pytest.mark.gpu
@pytest.mark.parametrize("kw", CONFIGS)
def test_stub_steps_like_the_oracle(kw):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from oracle import oracle as O
    stub = mirror_stub()
    cfg = C.EnvConfig(**kw)
    n = 257
    env = stub.B200BatchEnv(cfg, n, seed=5)
    ref = O.OracleBatchEnv(cfg, n, seed=5)
    assert np.array_equal(env.reset(), ref.reset())
    with pytest.raises(ValueError):
        env.step(np.full(n, cfg.n_actions))
    rng = np.random.default_rng(1)
    for t in range(30):
        a = rng.integers(0, cfg.n_actions, size=n)
        o1, r1, d1, i1 = env.step(a)
        o2, r2, d2, i2 = ref.step(a)
        assert np.array_equal(o1, o2) and np.array_equal(r1, r2) and np.array_equal(d1, d2), t
        assert all(np.array_equal(i1[k], i2[k]) for k in i2), t
