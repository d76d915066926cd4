"""c4 cost split: step kernel time with no-op actions (no recompute ever) vs
uniform random actions (about a third of the steps write and recompute)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

cfg = EnvConfig(domain="binary", max_width=64, max_height=64, obs_size=7)
n = 65536
env = BatchEnv(cfg, n, seed=0, validate=False)
obs = env.new_obs()
env.reset(out=obs)
r = torch.empty(n, dtype=torch.float64, device="cuda")
d = torch.empty(n, dtype=torch.bool, device="cuda")
K = 20
for label, mk in (("noop", lambda i: torch.zeros(n, dtype=torch.int64, device="cuda")),
                  ("random", lambda i: env.random_actions(i)),
                  ("all_write_wall", lambda i: torch.full((n,), 2, dtype=torch.int64, device="cuda"))):
    acts = [mk(i) for i in range(K)]
    for a in acts[:3]:
        env.step_raw(a, obs, r, d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for a in acts:
        env.step_raw(a, obs, r, d)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / K:.4f} ms/step")
