"""Split the fused c5 step into its phases (CUDA-event timed, 2^20 envs):
full step (logic + render + store), step without observation (logic only),
and observe (render + store only, no logic). Profiling helper; not a bench."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
dom = sys.argv[2] if len(sys.argv) > 2 else "binary"
env = BatchEnv(EnvConfig(domain=dom), n, seed=0, validate=False)
obs = env.new_obs()
env.reset(out=obs)
t = torch
rew = t.empty(n, dtype=t.float64, device="cuda")
done = t.empty(n, dtype=t.uint8, device="cuda")
acts = env.random_actions(1)


def timeit(fn, k=10):
    for i in range(3):
        fn(i)
    ev = [(t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)) for _ in range(k)]
    t.cuda.synchronize()
    tot = 0.0
    for i in range(k):
        env.random_actions(1000 + i, out=acts)
        ev[i][0].record()
        fn(i)
        ev[i][1].record()
    t.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / k


full = timeit(lambda i: env.step_raw(acts, obs, rew, done))
logic = timeit(lambda i: env.step_raw(acts, None, rew, done))
render = timeit(lambda i: env.observe(out=obs))
print(f"{dom} n={n}: full {full:.4f} ms  logic-only {logic:.4f} ms  observe-only {render:.4f} ms  "
      f"sum {logic + render:.4f} ms  -> {n / full / 1e3:.1f} M env-steps/s")
