"""One TrunkPolicy collect_rollout (c5 shape, 65,536 envs, 4 steps) for an
ncu launch list of its kernels: python tools/rollout_trunk_launches.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402
from paper_2408_12525_b200.policy import TrunkPolicy, collect_rollout, default_arch, init_policy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cfg = EnvConfig(domain="binary")
env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
bits = env.reset()
shp = env.observation_shape
model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).cuda()
pol = TrunkPolicy(model, shp)
gen = torch.Generator(device="cuda").manual_seed(0)
batch, bits, _ = collect_rollout(pol, env, 2, gen, bits)  # warm-up
torch.cuda.synchronize()
batch, bits, _ = collect_rollout(pol, env, 4, gen, bits)
torch.cuda.synchronize()
