"""A/B of the chained random-policy step (lg_step_random) against
lg_random_actions + lg_step, CUDA-graph replay of K steps, per config/size.

python tools/chain_ab.py [--steps 20] [--configs c5:1048576,c5:131072,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402


def run(cfg, B, K, variant):
    os.environ["LG_NO_CHAIN"] = "1" if variant == "random_unchained" else "0"
    env = BatchEnv(cfg, B, seed=0, validate=False)
    obs = env.new_obs()
    acts = torch.empty(B, dtype=torch.int64, device="cuda")
    rew = torch.empty(B, dtype=torch.float64, device="cuda")
    done = torch.empty(B, dtype=torch.bool, device="cuda")
    info = env._info_buffers()
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    env.reset(out=obs)

    def step(i):
        if variant == "split":
            env.random_actions(i, out=acts)
            env.step_raw(acts, obs, rew, done, info, stats)
        else:
            env.step_random(i, obs, rew, done, info, stats, actions_out=acts)

    for i in range(5):
        step(i)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            step(100 + i)
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        best = ms if best is None else min(best, ms)
    del g
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--configs", default="c5:1048576,c5:524288,c5:262144,c5:131072,c3,c2,c4,c1")
    ap.add_argument("--variants", default="split,random_unchained,chained")
    a = ap.parse_args()
    for item in a.configs.split(","):
        name, _, n = item.partition(":")
        desc, kw, default_b = bench.CONFIGS[name]
        B = int(n) if n else default_b
        cfg = EnvConfig(**kw)
        row = {"config": name, "envs": B}
        for v in a.variants.split(","):
            ms = run(cfg, B, a.steps, v)
            row[v] = {"ms_per_step": round(ms, 5), "Menv_steps_per_s": round(B / ms / 1e3, 2)}
            torch.cuda.empty_cache()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
