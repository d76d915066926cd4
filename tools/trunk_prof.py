"""Cycle accounting of the trunk kernel (a -DTK_PROF build):
    nvcc ... -DTK_PROF -o variants/tkprof.so; LG_LIB_PATH=variants/tkprof.so python tools/trunk_prof.py
MMA issuer: [issue, wait A3F, wait W3F, wait ACE, wait C1F, -, -, total];
epilogue group g thread 0: [wait ACF, wait A3E, -, total]."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200 import _lib  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402
from paper_2408_12525_b200.policy import TrunkPolicy, default_arch, init_policy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfg = EnvConfig(domain="binary")
env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
bits = env.reset()
shp = env.observation_shape
model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).cuda()
pol = TrunkPolicy(model, shp)
for _ in range(3):
    pol(bits, n)
torch.cuda.synchronize()
nb = (n + 127) // 128
buf = np.zeros((nb, 16), dtype=np.int64)
lib = _lib.load()
lib.lg_trunk_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.lg_trunk_prof(buf.ctypes.data_as(ctypes.c_void_p), nb))
m = buf.mean(0)
print("issuer: other %.0f  wA3F %.0f  wW3F %.0f  wACE %.0f  wC1F %.0f  conv2-issue %.0f  fc-issue %.0f  total %.0f" % (m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7]))
print("epi0: wACF %.0f wA3E %.0f total %.0f | epi1: wACF %.0f wA3E %.0f total %.0f" % (m[8], m[9], m[10], m[12], m[13], m[14]))
