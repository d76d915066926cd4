"""c5 step launches without an observation (step logic only): ncu helper."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

n = 1 << 20
env = BatchEnv(EnvConfig(domain="binary"), n, seed=0, validate=False)
env.reset()
rew = torch.empty(n, dtype=torch.float64, device="cuda")
done = torch.empty(n, dtype=torch.uint8, device="cuda")
for i in range(4):
    env.step_raw(env.random_actions(i), None, rew, done)
torch.cuda.synchronize()
print("ok")
