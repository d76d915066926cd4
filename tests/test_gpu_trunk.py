"""The tensor-core policy trunk (tcgen05 + TMEM) against torch references
(needs a B200).

``TrunkPolicy`` = ``lg_conv1_bits`` (tile layout) + ``lg_policy_trunk``: the
default ConvPolicy (nets.py:150-183) from packed observation bits, bf16
operands with fp32 accumulation. Two references on the same observations:

* the reference model in float32 (TF32 off) -- bf16 tolerance: the largest
  logit/value error within 2% of the largest magnitude;
* the same function with bf16 rounding at the kernel's rounding points
  (conv1 output, weights, conv2 output) -- within 0.3%, which pins the
  kernel's indexing (taps, pixel order, layouts) rather than bf16 noise.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2408_12525_b200.config import EnvConfig  # noqa: E402
from paper_2408_12525_b200.env import BatchEnv, unpack_obs  # noqa: E402
from paper_2408_12525_b200.policy import (TrunkPolicy, collect_rollout, default_arch,  # noqa: E402
                                          init_policy)

pytestmark = pytest.mark.gpu


def _no_tf32():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


def _bf(x):
    return x.to(torch.bfloat16).float()


def emulated(model, obs):
    """ConvPolicy forward with the kernel's bf16 rounding points."""
    F = torch.nn.functional
    c1w, c2w, fc = model.trunk[0], model.trunk[2], model.trunk[5]
    h = _bf(torch.relu(F.conv2d(obs, c1w.weight, c1w.bias)))
    h = _bf(torch.relu(F.conv2d(h, _bf(c2w.weight), c2w.bias)))
    h = torch.relu(h.flatten(1) @ _bf(fc.weight).T + fc.bias)
    return model.policy_head(h), model.value_head(h).squeeze(-1)


CASES = [
    (dict(domain="binary"), 300, 0),                                  # obs 31 (c5 shape), ragged last tile
    (dict(domain="maze", representation="turtle"), 256, 1),           # 6 channels, 8 actions
    (dict(domain="dungeon", max_width=8, max_height=8, obs_size=15), 129, 2),  # P2 = 11: ragged column chunk
    (dict(domain="binary", max_width=5, max_height=5, obs_size=5), 40, 3),     # P2 = 1
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_trunk_matches_torch(case):
    _no_tf32()
    kw, n, seed = CASES[case]
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=seed, obs_dtype="bits")
    bits = env.reset()
    for t in range(3):
        bits, _, _, _ = env.step(env.random_actions(t))
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=seed).cuda()
    with torch.no_grad():  # a larger head so the logits are not all ~0
        model.policy_head.weight.mul_(50.0)
        model.policy_head.bias.uniform_(-0.1, 0.1)
        model.trunk[2].bias.uniform_(-0.1, 0.1)
        model.trunk[5].bias.uniform_(-0.1, 0.1)
    pol = TrunkPolicy(model, shp)
    lg, v = pol(bits, n)
    obs = unpack_obs(bits, n, shp)
    with torch.no_grad():
        rl, rv = model(obs)
        el, ev = emulated(model, obs)
    for got, ref, emu in ((lg, rl, el), (v, rv, ev)):
        scale = float(ref.abs().max())
        assert float((got - emu).abs().max()) <= 3e-3 * scale + 1e-5, (float((got - emu).abs().max()), scale)
        assert float((got - ref).abs().max()) <= 2e-2 * scale + 1e-5, (float((got - ref).abs().max()), scale)


def test_trunk_rollout_and_refresh():
    """collect_rollout (ppo.py:101-143) with the fused trunk; refresh() picks
    up new weights."""
    _no_tf32()
    cfg = EnvConfig(domain="binary")
    n = 4096
    env = BatchEnv(cfg, n, seed=0, validate=False, obs_dtype="bits")
    bits = env.reset()
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=0).cuda()
    pol = TrunkPolicy(model, shp)
    gen = torch.Generator(device="cuda").manual_seed(0)
    batch, bits2, _ = collect_rollout(pol, env, 4, gen, bits)
    assert batch.actions.shape == (4, n) and int(batch.actions.max()) < cfg.n_actions
    assert env.errors() == 0
    with torch.no_grad():
        model.policy_head.bias.add_(1.0)
    l0, _ = pol(bits2, n)
    pol.refresh()
    l1, _ = pol(bits2, n)
    assert torch.allclose(l1 - l0, torch.ones_like(l0), atol=1e-4)


def _tiles_to_nhwc(tiles, n, P1):
    """[tile][px][2048] UMMA core-matrix blocks -> [n, px, 16] (trunk_kernel.cuh layout)."""
    NP = P1 * P1
    t = tiles.float().view(-1, NP, 2, 16, 8, 8)  # tile, px, h, m>>3, m&7, channel
    return t.permute(0, 3, 4, 1, 2, 5).reshape(-1, NP, 16)[:n]


@pytest.mark.parametrize("kw,n", [(dict(domain="binary"), 300),
                                  (dict(domain="binary", max_width=5, max_height=5, obs_size=5), 40),
                                  (dict(domain="binary", max_width=12, max_height=12, obs_size=9), 1000)])
def test_conv1_row_triple_tiles(kw, n, monkeypatch):
    """The row-triple conv1 (C <= 2) against the float32 conv and the
    generic table kernel (LG_CONV1_GENERIC=1), same tile layout."""
    _no_tf32()
    cfg = EnvConfig(**kw)
    env = BatchEnv(cfg, n, seed=7, obs_dtype="bits")
    bits = env.reset()
    for t in range(4):
        bits, _, _, _ = env.step(env.random_actions(t))
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=1).cuda()
    with torch.no_grad():
        model.trunk[0].bias.uniform_(-0.2, 0.2)
    pol = TrunkPolicy(model, shp)
    tri = _tiles_to_nhwc(pol.conv1_tiles(bits, n), n, pol.P1)
    monkeypatch.setenv("LG_CONV1_GENERIC", "1")
    gen = _tiles_to_nhwc(pol.conv1_tiles(bits, n), n, pol.P1)
    obs = unpack_obs(bits, n, shp)
    c1 = model.trunk[0]
    with torch.no_grad():
        ref = torch.relu(torch.nn.functional.conv2d(obs, c1.weight, c1.bias))
    ref = ref.permute(0, 2, 3, 1).reshape(n, -1, 16)
    # fp16 row tables (policy_kernels.cuh): within a bfloat16 ulp of the
    # float32 conv, plus 1e-3 of the largest activation for cancellation
    scale = float(ref.abs().max())
    assert torch.allclose(tri, gen, rtol=8e-3, atol=1e-3 * scale)
    assert torch.allclose(tri, _bf(ref), rtol=8e-3, atol=1e-3 * scale)
    assert float((tri - ref).abs().max()) <= 8e-3 * scale


def test_conv1_row_triple_non_onehot_bits(monkeypatch):
    """Arbitrary bits (cells that are not one-hot) take the nine-tap path of
    the row-triple kernel and still equal the generic kernel."""
    _no_tf32()
    cfg = EnvConfig(domain="binary")
    n = 96
    shp = cfg.observation_shape
    words = (n * shp[0] * shp[1] * shp[2] + 31) // 32
    g = torch.Generator(device="cuda").manual_seed(3)
    bits = torch.randint(-2 ** 31, 2 ** 31 - 1, (words,), dtype=torch.int32, device="cuda", generator=g)
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=2).cuda()
    pol = TrunkPolicy(model, shp)
    tri = _tiles_to_nhwc(pol.conv1_tiles(bits, n), n, pol.P1)
    monkeypatch.setenv("LG_CONV1_GENERIC", "1")
    gen = _tiles_to_nhwc(pol.conv1_tiles(bits, n), n, pol.P1)
    assert torch.allclose(tri, gen, rtol=8e-3, atol=1e-6)


def test_trunk_fused_sampling():
    """lg_policy_trunk_sample: the same logits/value as lg_policy_trunk, the
    log-probability of the drawn action, and draws distributed as
    softmax(logits) (ppo.py:125-130)."""
    _no_tf32()
    cfg = EnvConfig(domain="maze", representation="turtle")  # 8 actions
    n = 16384
    env = BatchEnv(cfg, n, seed=1, obs_dtype="bits")
    bits = env.reset()
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=4).cuda()
    with torch.no_grad():
        model.policy_head.weight.mul_(20.0)
        model.policy_head.bias.uniform_(-1.0, 1.0)
    pol = TrunkPolicy(model, shp)
    a, lp, v, lg = pol.sample(bits, n, seed=5)
    l0, v0 = pol(bits, n)
    assert torch.equal(lg, l0) and torch.equal(v, v0)
    assert int(a.min()) >= 0 and int(a.max()) < cfg.n_actions
    ref_lp = torch.log_softmax(lg, -1).gather(1, a[:, None]).squeeze(1)
    assert torch.allclose(lp, ref_lp, atol=1e-4, rtol=1e-4)
    probs = torch.softmax(lg, -1)
    freq = torch.nn.functional.one_hot(a, cfg.n_actions).float().mean(0)
    assert float((freq - probs.mean(0)).abs().max()) < 0.02
    a2, _, _, _ = pol.sample(bits, n, seed=5)
    a3, _, _, _ = pol.sample(bits, n, seed=6)
    assert torch.equal(a, a2) and not torch.equal(a, a3)


@pytest.mark.parametrize("n", [300, 128 * 158 + 5])
def test_trunk_tail_split_pairs(n, monkeypatch):
    """The tiles past the last whole wave run as half-tile CTA pairs (FC
    partials summed through DSMEM): the same logits/value as whole tiles
    (LG_TRUNK_TAIL=0) up to fp32 summation order, and the torch reference."""
    _no_tf32()
    cfg = EnvConfig(domain="binary")
    env = BatchEnv(cfg, n, seed=2, obs_dtype="bits")
    bits = env.reset()
    bits, _, _, _ = env.step(env.random_actions(1))
    shp = env.observation_shape
    model = init_policy(default_arch(shp[1], shp[0], cfg.n_actions), seed=3).cuda()
    with torch.no_grad():
        model.policy_head.weight.mul_(50.0)
        model.trunk[5].bias.uniform_(-0.1, 0.1)
    pol = TrunkPolicy(model, shp)
    lg, v = pol(bits, n)
    monkeypatch.setenv("LG_TRUNK_TAIL", "0")
    lg0, v0 = pol(bits, n)
    for a, b in ((lg, lg0), (v, v0)):
        scale = float(b.abs().max())
        assert float((a - b).abs().max()) <= 1e-4 * scale + 1e-5  # fp32 sums of ~23k terms, reordered
    obs = unpack_obs(bits, n, shp)
    with torch.no_grad():
        el, ev = emulated(model, obs)
    for got, emu in ((lg, el), (v, ev)):
        scale = float(emu.abs().max())
        assert float((got - emu).abs().max()) <= 3e-3 * scale + 1e-5
