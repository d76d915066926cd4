"""Cost of a lockstep reset step (every env finishes and auto-resets at once),
with and without the episode-stats accumulation: python tools/reset_step.py [n_envs]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
L = 16
for with_stats in (True, False):
    cfg = EnvConfig(domain="binary", max_steps=L)
    env = BatchEnv(cfg, n, seed=0, validate=False)
    obs = env.new_obs()
    rew = torch.empty(n, dtype=torch.float64, device="cuda")
    done = torch.empty(n, dtype=torch.bool, device="cuda")
    info = env._info_buffers()
    stats = torch.zeros(5, dtype=torch.float64, device="cuda") if with_stats else None
    acts = torch.empty(n, dtype=torch.int64, device="cuda")
    env.reset(out=obs)
    ev = []
    for i in range(3 * L):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        env.random_actions(i, out=acts)
        a.record()
        env.step_raw(acts, obs, rew, done, info, stats)
        b.record()
        ev.append((i + 1, a, b))
    torch.cuda.synchronize()
    t = {k: a.elapsed_time(b) for k, a, b in ev}
    resets = [t[k] for k in t if k % L == 0 and k > L]
    steady = sorted(t[k] for k in t if k % L and k > L)
    print(json.dumps({"envs": n, "stats": with_stats, "reset_step_ms": resets,
                      "steady_median_ms": steady[len(steady) // 2]}))
    del env, obs
    torch.cuda.empty_cache()
