"""c5 observe-only launches (render + write, no step logic): ncu helper."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

env = BatchEnv(EnvConfig(domain="binary"), 1 << 20, seed=0, validate=False)
obs = env.new_obs()
env.reset(out=obs)
for _ in range(4):
    env.observe(out=obs)
torch.cuda.synchronize()
print("ok")
