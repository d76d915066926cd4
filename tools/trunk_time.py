"""Time the tensor-core policy trunk on the c5 observation shape:
python tools/trunk_time.py [n_envs]

Prints the two kernels' times (lg_conv1_bits tile layout, lg_policy_trunk),
the trunk's achieved tensor throughput (algorithmic conv2 + FC flops) and the
collect_rollout rate with TrunkPolicy vs PackedPolicy (conv1_bits + torch)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402
from paper_2408_12525_b200.policy import (PackedPolicy, TrunkPolicy, collect_rollout,  # noqa: E402
                                          default_arch, init_policy)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
cfg = EnvConfig(domain="binary")
env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
bits = env.reset()
shp = env.observation_shape
model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).cuda()
pol = TrunkPolicy(model, shp)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


c1 = pol.conv1_tiles(bits, n)
t_c1 = timed(lambda: pol.conv1_tiles(bits, n))
na = cfg.n_actions
lg = torch.empty((n, na), device="cuda")
v = torch.empty(n, device="cuda")
import ctypes  # noqa: E402

from paper_2408_12525_b200 import _lib  # noqa: E402

p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def trunk():
    _lib.check(_lib.load().lg_policy_trunk(p(c1), n, pol.P1, p(pol.w2), p(pol.b2), p(pol.w3), p(pol.b3), p(pol.wh),
                                           p(pol.bh), na, p(lg), p(v),
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


t_tr = timed(trunk)
P1 = shp[1] - 2
P2 = P1 - 2
flops = n * (P2 * P2 * 32 * 144 * 2 + 32 * P2 * P2 * 64 * 2)
out = {"envs": n, "conv1_tiles_ms": t_c1, "conv1_out_gbs": c1.numel() * 2 / t_c1 / 1e6,
       "trunk_ms": t_tr, "trunk_tflops": flops / t_tr / 1e9}


def rate(make, steps=8):
    e = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
    o = e.reset()
    pp = make()
    gen = torch.Generator(device="cuda").manual_seed(0)
    _, o, _ = collect_rollout(pp, e, 2, gen, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    collect_rollout(pp, e, steps, gen, o)
    e1.record()
    torch.cuda.synchronize()
    return n * steps / (e0.elapsed_time(e1) / 1e3)


out["rollout_tcgen05_trunk"] = rate(lambda: pol)
out["rollout_conv1_bits_torch_bf16"] = rate(lambda: PackedPolicy(model, shp, bf16=True))
print(json.dumps(out))
