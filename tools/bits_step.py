import torch, sys, os
sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig
from paper_2408_12525_b200.env import BatchEnv
n = 65536
for fmt in ("bits", "float32"):
    env = BatchEnv(EnvConfig(domain="binary"), n, seed=0, validate=False, obs_dtype=fmt)
    obs = env.new_obs(); env.reset(out=obs)
    rew = torch.empty(n, dtype=torch.float64, device="cuda"); done = torch.empty(n, dtype=torch.bool, device="cuda")
    acts = [env.random_actions(i) for i in range(20)]
    for i in range(5): env.step_raw(acts[i], obs, rew, done)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): env.step_raw(acts[i], obs, rew, done)
    e1.record(); torch.cuda.synchronize()
    print(fmt, os.environ.get("LG_FORCE_TEAM", "0"), "%.1f us/step" % (e0.elapsed_time(e1) / 20 * 1e3))
