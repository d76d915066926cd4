"""Policy consumer on the GPU: packed observations and the
fused first conv (lg_conv1_bits) against torch on the unpacked float32 planes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv, unpack_obs  # noqa: E402
from paper_2408_12525_b200.policy import (PackedPolicy, collect_rollout, conv1_bits, default_arch,  # noqa: E402
                                          init_policy)

pytestmark = pytest.mark.gpu
F = torch.nn.functional

CASES = [
    (dict(domain="binary"), 20000),                                          # c5 shape, solo warp + elided plane
    (dict(domain="binary"), 64),                                             # c1: block mode, shared words
    (dict(domain="maze", representation="turtle"), 4096),                    # c2: lane team 16
    (dict(domain="dungeon", representation="wide", pinpoints=("player", "key", "door"),
          randomize_shape=True), 20000),                                     # c3: stream layout
    (dict(domain="binary", max_width=64, max_height=64, obs_size=7), 700),   # c4 shape: lane team 64
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_bits_env_equals_float32_env(case):
    kw, n = CASES[case]
    cfg = EnvConfig(**kw)
    f32 = BatchEnv(cfg, n, seed=3, validate=False)
    bits = BatchEnv(cfg, n, seed=3, validate=False, obs_dtype="bits")
    a, b = f32.reset(), bits.reset()
    assert b.dtype == torch.int32 and b.numel() == (a.numel() + 31) // 32
    assert torch.equal(unpack_obs(b, n, f32.observation_shape), a)
    for t in range(4):
        acts = f32.random_actions(100 + t)
        a, ra, da, _ = f32.step(acts)
        b, rb, db, _ = bits.step(acts)
        assert torch.equal(unpack_obs(b, n, f32.observation_shape), a), t
        assert torch.equal(ra, rb) and torch.equal(da, db), t


@pytest.mark.parametrize("K", [16, 17, 32, 64])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_conv1_bits_matches_conv2d(case, K):
    kw, n = CASES[case]
    n = min(n, 3000)
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=5, validate=False, obs_dtype="bits")
    bits = env.reset()
    for t in range(3):
        bits = env.step(env.random_actions(t))[0]
    shape = env.observation_shape
    obs = unpack_obs(bits, n, shape)
    g = torch.Generator(device="cuda").manual_seed(K)
    w = torch.randn((K, shape[0], 3, 3), device="cuda", generator=g)
    b = torch.randn(K, device="cuda", generator=g)
    # float64 reference (cuDNN's float32 path may use TF32); the kernel sums
    # at most 9 * ceil(C/4) + 1 float32 table entries per output
    lin64 = F.conv2d(obs.double(), w.double(), b.double())
    want = F.relu(lin64).float()
    got = conv1_bits(bits, n, shape, w, b)
    torch.testing.assert_close(got, want, rtol=1e-5, atol=1e-5)
    got16 = conv1_bits(bits, n, shape, w, b, out_dtype=torch.bfloat16)
    torch.testing.assert_close(got16.float(), want, rtol=1e-2, atol=1e-2)
    lin = conv1_bits(bits, n, shape, w, b, relu=False)
    torch.testing.assert_close(lin, lin64.float(), rtol=1e-5, atol=1e-5)
    # channels-last output: the same tensor values, NHWC strides
    cl = conv1_bits(bits, n, shape, w, b, channels_last=True)
    assert cl.stride(1) == 1 and torch.equal(cl, got)
    cl16 = conv1_bits(bits, n, shape, w, b, out_dtype=torch.bfloat16, channels_last=True)
    assert torch.equal(cl16, got16)


@pytest.fixture(autouse=True)
def _no_tf32():
    prev = torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32
    torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = prev


def test_packed_policy_matches_conv_policy():
    cfg = EnvConfig(domain="binary")
    n = 4096
    env = BatchEnv(cfg, n, seed=1, validate=False, obs_dtype="bits")
    bits = env.reset()
    shape = env.observation_shape
    model = init_policy(default_arch(shape[1], shape[0], cfg.n_actions), seed=0).cuda()
    with torch.no_grad():
        l1, v1 = model(unpack_obs(bits, n, shape))
        l2, v2 = PackedPolicy(model, shape)(bits, n)
        l3, v3 = PackedPolicy(model, shape, channels_last=True)(bits, n)
    torch.testing.assert_close(l2, l1, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(v2, v1, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(l3, l1, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(v3, v1, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("packed", [False, True])
def test_collect_rollout_replays_through_the_env(packed):
    """The rollout's actions, replayed through a fresh env with the same seed,
    give the recorded rewards, dones and observations (ppo.py:101-143 bookkeeping)."""
    cfg = EnvConfig(domain="binary", max_width=8, max_height=8, obs_size=9, max_steps=15)
    n, T = 512, 40
    fmt = "bits" if packed else "float32"
    env = BatchEnv(cfg, n, seed=7, validate=False, obs_dtype=fmt)
    shape = env.observation_shape
    model = init_policy(default_arch(shape[1], shape[0], cfg.n_actions), seed=3).cuda()
    pol = PackedPolicy(model, shape) if packed else model
    gen = torch.Generator(device="cuda").manual_seed(11)
    obs0 = env.reset()
    batch, last, finished = collect_rollout(pol, env, T, gen, obs0)
    assert batch.actions.shape == (T, n) and batch.rewards.dtype == torch.float64
    ref = BatchEnv(cfg, n, seed=7, validate=False)
    o = ref.reset()
    ep = []
    for t in range(T):
        seen = batch.obs[t]
        assert torch.equal(unpack_obs(seen, n, shape) if packed else seen, o), t
        o, r, d, info = ref.step(batch.actions[t])
        assert torch.equal(r, batch.rewards[t]) and torch.equal(d, batch.dones[t]), t
        ep += info["episode_reward"][d].tolist()
    assert finished == ep
    assert torch.equal(unpack_obs(last, n, shape) if packed else last, o)
    # logprobs are the policy's log-softmax at the taken actions
    with torch.no_grad():
        x = unpack_obs(batch.obs[0], n, shape) if packed else batch.obs[0]
        logits, value = model(x)
        lp = torch.log_softmax(logits, -1).gather(1, batch.actions[0][:, None]).squeeze(1)
    torch.testing.assert_close(batch.logprobs[0], lp, rtol=1e-4, atol=1e-5)
    torch.testing.assert_close(batch.values[0], value, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("case", [0, 2, 4])
def test_numpy_env_bits_format(case):
    """NumpyBatchEnv(obs_dtype="bits") returns the packed stream itself (lg_step_host, no expansion)."""
    from paper_2408_12525_b200.env import NumpyBatchEnv
    kw, n = CASES[case]
    n = min(n, 5000)
    cfg = EnvConfig(**kw)
    dev = BatchEnv(cfg, n, seed=8, validate=False, obs_dtype="bits")
    host = NumpyBatchEnv(cfg, n, seed=8, obs_dtype="bits")
    assert np.array_equal(dev.reset().cpu().numpy(), host.reset())
    rng = np.random.default_rng(case)
    for t in range(3):
        a = rng.integers(0, cfg.n_actions, size=n)
        o1, r1, _, _ = dev.step(torch.from_numpy(a).cuda())
        o2, r2, _, _ = host.step(a)
        assert o2.dtype == np.int32 and np.array_equal(o1.cpu().numpy(), o2), t
        assert np.array_equal(r1.cpu().numpy(), r2), t


def test_conv1_bits_large_window_and_bad_arguments():
    """A 64x64 dungeon window of 96 (C=8): four observations' masks + bits do not
    fit in shared memory, so the kernel takes fewer envs per iteration."""
    from paper_2408_12525_b200 import _lib
    cfg = EnvConfig(domain="dungeon", max_width=64, max_height=64, obs_size=95)
    n = 40
    env = BatchEnv(cfg, n, seed=2, validate=False, obs_dtype="bits")
    bits = env.reset()
    shape = env.observation_shape
    obs = unpack_obs(bits, n, shape)
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn((16, shape[0], 3, 3), device="cuda", generator=g)
    b = torch.randn(16, device="cuda", generator=g)
    want = F.relu(F.conv2d(obs.double(), w.double(), b.double())).float()
    torch.testing.assert_close(conv1_bits(bits, n, shape, w, b), want, rtol=1e-5, atol=1e-5)
    with pytest.raises(ValueError):
        conv1_bits(bits, n, shape, torch.zeros((65, shape[0], 3, 3), device="cuda"), torch.zeros(65, device="cuda"))
    with pytest.raises(ValueError):
        _lib.check(_lib.load().lg_conv1_bits(None, n, shape[0], shape[1], shape[2], None, None, 16, None, 0, 1, 0,
                                             None))
