"""Helpers to load the golden fixtures written by tests/golden/make_golden.py."""
from __future__ import annotations

import ast
import glob
import hashlib
import os

import numpy as np

from paper_2408_12525_b200.config import EnvConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def env_case_names() -> list[str]:
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "env_*.npz")))


def load_env_case(name: str):
    z = np.load(os.path.join(GOLDEN, f"env_{name}.npz"))
    kw = ast.literal_eval(str(z["config"]))
    rep = str(z["representation"])
    cfg = EnvConfig(**kw, representation=rep)
    return cfg, z


def load(name: str):
    return np.load(os.path.join(GOLDEN, name))
