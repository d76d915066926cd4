"""Check a kernel variant (env vars set by the caller) against the default path."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CODE = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, "%s")
from paper_2408_12525_b200.config import EnvConfig
from paper_2408_12525_b200.env import BatchEnv
cfg = EnvConfig(domain=sys.argv[1])
n = int(sys.argv[2])
env = BatchEnv(cfg, n, seed=3)
h = hashlib.sha256()
h.update(env.reset().cpu().numpy().tobytes())
for t in range(6):
    a = env.random_actions(t)
    o, r, d, _ = env.step(a)
    h.update(o.cpu().numpy().tobytes()); h.update(r.cpu().numpy().tobytes())
print(h.hexdigest())
''' % ROOT

for domain in ("binary", "maze", "dungeon"):
    outs = []
    for extra in ({}, dict(os.environ)):
        env = dict(os.environ)
        if not extra:
            env.pop("LG_WS", None)
        r = subprocess.run([sys.executable, "-c", CODE, domain, "40000"], capture_output=True, text=True, env=env)
        outs.append(r.stdout.strip() or r.stderr[-500:])
    print(domain, "MATCH" if outs[0] == outs[1] else f"MISMATCH {outs}")
