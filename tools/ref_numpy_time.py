"""The reference's own numpy BatchEnv timed in the build container (it reads
/root/reference, so it never runs on the GPU box): python tools/ref_numpy_time.py"""
import sys, time
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
from levelgen.env import BatchEnv, EnvConfig
cfg = EnvConfig(domain="binary")
n = 4096
env = BatchEnv(cfg, n, seed=0)
env.reset()
rng = np.random.default_rng(1)
acts = [rng.integers(0, cfg.n_actions, size=n) for _ in range(13)]
for a in acts[:3]: env.step(a)
t0 = time.perf_counter()
for a in acts[3:]: env.step(a)
dt = time.perf_counter() - t0
print(f"reference numpy BatchEnv, binary16 obs31, {n} envs x 10 steps, 1 process: {n*10/dt:.0f} env-steps/s")
