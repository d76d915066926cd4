"""Small invocations of every kernel family, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py

Each case steps a few envs through one launch shape and checks the result
against the CPU oracle, so a run that the sanitizer passes is also correct:
solo block mode (cooperative render), solo warp mode with the per-env slot
layout and with the warp-wide bit stream (shared-memory atomicOr merges),
specialised and generic kernels, the lane-team kernels of 16/32/64 rows (union
-find with 16-bit CAS in shared memory), the packed host transfer, state
export/import, the metrics kernel, and the policy kernels (conv1_bits and the
tcgen05 trunk)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv, NumpyBatchEnv, unpack_obs  # noqa: E402
from paper_2408_12525_b200.policy import TrunkPolicy, conv1_bits, default_arch, init_policy  # noqa: E402

CASES = [
    ("solo block (c1)", dict(domain="binary"), 64, {}),
    ("solo warp slot + elided frozen", dict(domain="binary"), 4736 * 4, {}),
    ("solo warp stream (c3 spec, early)", dict(domain="dungeon", representation="wide",
                                               pinpoints=("player", "key", "door"), randomize_shape=True), 4736 * 4, {}),
    ("solo warp generic", dict(domain="binary", change_budget=2), 4736 * 4, {"LG_NO_SPEC": "1"}),
    ("team 16 spec (c2)", dict(domain="maze", representation="turtle"), 2048, {}),
    ("team 16 generic ctrl", dict(domain="maze", controllable=("path_length",)), 2048, {}),
    ("team 32", dict(domain="dungeon", max_width=40, max_height=20, obs_size=33,
                     pinpoints=("player", "key", "door")), 257, {}),
    ("team 64 spec (c4)", dict(domain="binary", max_width=64, max_height=64, obs_size=7), 128, {}),
]


def run_case(name, kw, n, env_vars, steps=3):
    for k, v in env_vars.items():
        os.environ[k] = v
    try:
        cfg = EnvConfig(**kw)
        env = BatchEnv(cfg, n, seed=3)
        ref = O.OracleBatchEnv(cfg, n, seed=3)
        assert np.array_equal(env.reset().cpu().numpy(), ref.reset()), name
        rng = np.random.default_rng(7)
        for t in range(steps):
            a = rng.integers(0, cfg.n_actions, size=n)
            o1, r1, d1, _ = env.step(a)
            o2, r2, d2, _ = ref.step(a)
            assert np.array_equal(r1.cpu().numpy(), r2), (name, t)
            assert np.array_equal(o1.cpu().numpy(), o2), (name, t)
        sd = env.state_dict()
        twin = BatchEnv(cfg, n, seed=99)
        twin.load_state_dict(sd)
        assert np.array_equal(twin.observe().cpu().numpy(), env.observe().cpu().numpy()), name
    finally:
        for k in env_vars:
            os.environ.pop(k, None)
    print("ok", name, flush=True)


def main():
    for c in CASES:
        run_case(*c)
    # packed host transfer (bit stream + host expansion)
    os.environ["LG_HOST_EXPAND"] = "1"
    cfg = EnvConfig(domain="binary")
    host = NumpyBatchEnv(cfg, 300, seed=1, copy=False)
    ref = O.OracleBatchEnv(cfg, 300, seed=1)
    host.reset()
    ref.reset()
    a = np.random.default_rng(0).integers(0, 3, size=300)
    assert np.array_equal(host.step(a)[0], ref.step(a)[0])
    os.environ.pop("LG_HOST_EXPAND")
    print("ok packed host transfer", flush=True)
    # policy kernels
    env = BatchEnv(cfg, 200, seed=0, obs_dtype="bits")
    bits = env.reset()
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).cuda()
    c1 = conv1_bits(bits, 200, shp, model.trunk[0].weight, model.trunk[0].bias)
    ref1 = torch.relu(torch.nn.functional.conv2d(unpack_obs(bits, 200, shp), model.trunk[0].weight,
                                                 model.trunk[0].bias))
    assert float((c1 - ref1).detach().abs().max()) < 1e-4
    lg, v = TrunkPolicy(model, shp)(bits, 200)
    torch.cuda.synchronize()
    assert torch.isfinite(lg).all() and torch.isfinite(v).all()
    print("ok policy kernels", flush=True)


if __name__ == "__main__":
    main()
