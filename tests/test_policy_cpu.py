"""Policy mirror (paper_2408_12525_b200.policy) vs the reference's nets.py,
pinned by tests/golden/policy.npz (made from the live reference by
tests/golden/make_policy_golden.py): same parameter names, shapes, counts and
seeded initial weights, and the same forward pass (CPU, float32)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2408_12525_b200.policy import ArchConfig, count_params, default_arch, init_policy  # noqa: E402

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "policy.npz"))
ARCHS = [
    (7, 4, 3, (16, 32), (64,), 0),
    (9, 6, 8, (16, 32), (64,), 5),
    (4, 4, 3, (16,), (64,), 1),
    (11, 8, 768, (8, 12), (16, 8), 2),
]


@pytest.mark.parametrize("i", range(len(ARCHS)))
def test_init_and_forward_match_reference(i):
    o, c, a, cc, fc, seed = ARCHS[i]
    arch = ArchConfig(o, c, a, cc, fc)
    assert count_params(arch) == int(GOLD[f"a{i}_count"])
    model = init_policy(arch, seed)
    sd = model.state_dict()
    want = {k.split("/", 1)[1]: GOLD[k] for k in GOLD.files if k.startswith(f"a{i}_param/")}
    assert sorted(sd) == sorted(want)
    for k, v in want.items():
        assert np.array_equal(sd[k].numpy(), v), k
    with torch.no_grad():
        logits, value = model(torch.from_numpy(GOLD[f"a{i}_obs"]))
    np.testing.assert_allclose(logits.numpy(), GOLD[f"a{i}_logits"], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(value.numpy(), GOLD[f"a{i}_value"], rtol=1e-6, atol=1e-6)


def test_arch_validation_and_defaults():
    assert default_arch(3, 4, 3).conv_channels == (16,)
    assert default_arch(31, 4, 3).conv_channels == (16, 32)
    with pytest.raises(ValueError):
        ArchConfig(3, 4, 3, (16, 32), (64,))
    with pytest.raises(ValueError):
        ArchConfig(7, 4, 1)
    with pytest.raises(ValueError):
        init_policy(ArchConfig(7, 4, 3), 0)(torch.zeros(2, 4, 5, 5))


def test_trunk_weight_packing_layouts():
    """pack_conv2_weight / pack_fc_weight put element (n, k) of each block at
    ((k/8)*(N/8) + n/8)*64 + (n%8)*8 + k%8 (UMMA K-major core matrices,
    csrc/trunk_kernel.cuh); conv2 blocks hold three taps side by side (N = 96)."""
    import torch
    from paper_2408_12525_b200.policy import pack_conv2_weight, pack_fc_weight
    w2 = torch.randn(32, 16, 3, 3)
    p2 = pack_conv2_weight(w2).float()
    side = 5
    w3 = torch.randn(64, 32 * side * side)
    p3 = pack_fc_weight(w3, 32, side).float()
    g = torch.Generator().manual_seed(0)
    for _ in range(200):
        t, n, k = (int(torch.randint(9, (1,), generator=g)), int(torch.randint(32, (1,), generator=g)),
                   int(torch.randint(16, (1,), generator=g)))
        dy, dx = t // 3, t % 3
        nn = (2 - dx) * 32 + n  # taps (dy, 2), (dy, 1), (dy, 0) side by side: N = 96
        off = ((k // 8) * 12 + nn // 8) * 64 + (nn % 8) * 8 + k % 8
        assert p2[dy, off] == w2[n, k, dy, dx].bfloat16().float()
        px, n, k = (int(torch.randint(side * side, (1,), generator=g)), int(torch.randint(64, (1,), generator=g)),
                    int(torch.randint(32, (1,), generator=g)))
        off = ((k // 8) * 8 + n // 8) * 64 + (n % 8) * 8 + k % 8
        assert p3[px, off] == w3[n, k * side * side + px].bfloat16().float()
