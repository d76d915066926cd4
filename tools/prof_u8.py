"""Run a few uint8-observation steps (profiling helper for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
env = BatchEnv(EnvConfig(domain="binary"), n, seed=0, validate=False, obs_dtype="uint8")
env.reset()
for t in range(5):
    env.step(env.random_actions(t))
torch.cuda.synchronize()
print("ok")
