"""c3 in steady state with and without episode ends in the timed window
(max_steps raised so no env resets): what the reset path costs.
python tools/c3_resets.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

n, K = 65536, 40
for ms in (None, 100000):
    cfg = EnvConfig(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
                    randomize_shape=True, max_steps=ms)
    env = BatchEnv(cfg, n, seed=0, validate=False)
    obs = env.new_obs()
    rew = torch.empty(n, dtype=torch.float64, device="cuda")
    done = torch.empty(n, dtype=torch.bool, device="cuda")
    acts = torch.empty(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    env.reset(out=obs)
    for i in range(400):  # burn-in: with the default max_steps most envs have reset by now
        env.step_random(i, obs, rew, done, None, stats, actions_out=acts)
    torch.cuda.synchronize()
    before = float(stats[0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        env.step_random(1000 + i, obs, rew, done, None, stats, actions_out=acts)
    e1.record()
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / K
    print(json.dumps({"max_steps": ms, "ms_per_step": round(ms_step, 4), "Menv_steps_per_s": round(n / ms_step / 1e3, 1),
                      "episodes_in_window": float(stats[0]) - before}))
    del env
    torch.cuda.empty_cache()
