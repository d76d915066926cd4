"""Time lg_conv1_bits on a c5-shaped batch (binary 16x16, obs 31, K=16) and the
float32 cuDNN conv for contrast: python tools/conv1_time.py [n_envs]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv, unpack_obs  # noqa: E402
from paper_2408_12525_b200.policy import conv1_bits  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
for kw in (dict(domain="binary"), dict(domain="dungeon", representation="wide")):
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
    bits = env.reset()
    shp = env.observation_shape
    w = torch.randn(16, shp[0], 3, 3, device="cuda")
    b = torch.randn(16, device="cuda")
    for dt in (torch.float32, torch.bfloat16):
        out = conv1_bits(bits, n, shp, w, b, out_dtype=dt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            conv1_bits(bits, n, shp, w, b, out_dtype=dt, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gb = out.numel() * out.element_size() / ms / 1e6
        print(f"{cfg.domain} {shp} {dt}: {ms:.3f} ms  {gb:.0f} GB/s (output)")
