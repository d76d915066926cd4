"""Break one packed-policy rollout step into its parts (c5 config, 65,536 envs):
python tools/rollout_prof.py [n_envs] [benchmark 0/1] [channels_last 0/1]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv  # noqa: E402
from paper_2408_12525_b200.policy import conv1_bits, default_arch, init_policy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
torch.backends.cudnn.benchmark = len(sys.argv) > 2 and sys.argv[2] == "1"
cl = len(sys.argv) > 3 and sys.argv[3] == "1"
cfg = EnvConfig(domain="binary")
env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
bits = env.reset()
shp = env.observation_shape
model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), 0).cuda()
if cl:
    model = model.to(memory_format=torch.channels_last)
conv, rest = model.trunk[0], model.trunk[2:]
gen = torch.Generator(device="cuda").manual_seed(0)


def t(name, fn, reps=5):
    r = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        r = fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / reps:8.3f} ms")
    return r


with torch.no_grad():
    h1 = t("conv1_bits bf16", lambda: conv1_bits(bits, n, shp, conv.weight, conv.bias, out_dtype=torch.bfloat16))
    if cl:
        h1 = h1.contiguous(memory_format=torch.channels_last)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        c2 = model.trunk[2]
        h2 = t("conv2+relu (bf16)", lambda: torch.relu(c2(h1)))
        h3 = t("flatten+fc+relu (bf16)", lambda: model.trunk[5](model.trunk[4](h2.flatten(1) if not cl else h2.contiguous().flatten(1))))
        lg = t("heads (bf16)", lambda: (model.policy_head(h3), model.value_head(h3)))[0]
    p = torch.softmax(lg.float(), -1)
    a = t("multinomial", lambda: torch.multinomial(p, 1, generator=gen).squeeze(1))
    t("log_softmax+gather", lambda: torch.log_softmax(lg.float(), -1).gather(1, a[:, None]))
    t("env.step (bits)", lambda: env.step(a))
