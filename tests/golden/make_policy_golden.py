"""Golden fixtures for the policy consumer, from the LIVE reference (build container only):

    python tests/golden/make_policy_golden.py

Writes policy.npz: for a few small architectures, the reference's
``nets.init_policy(arch, seed)`` parameters (nets.py:186-189), its
``count_params`` and its forward pass on fixed 0/1 observations."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/reference/pkg/src")
from levelgen import nets  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ARCHS = [  # (obs_size, in_channels, n_actions, conv_channels, fc_dims, seed)
    (7, 4, 3, (16, 32), (64,), 0),
    (9, 6, 8, (16, 32), (64,), 5),
    (4, 4, 3, (16,), (64,), 1),
    (11, 8, 768, (8, 12), (16, 8), 2),
]


def main():
    out = {}
    for i, (o, c, a, cc, fc, seed) in enumerate(ARCHS):
        arch = nets.ArchConfig(obs_size=o, in_channels=c, n_actions=a, conv_channels=cc, fc_dims=fc)
        model = nets.init_policy(arch, seed)
        out[f"a{i}_count"] = np.array(nets.count_params(arch))
        for k, v in model.state_dict().items():
            out[f"a{i}_param/{k}"] = v.numpy()
        x = (np.random.default_rng(i).random((5, c, o, o)) < 0.5).astype(np.float32)
        with torch.no_grad():
            logits, value = model(torch.from_numpy(x))
        out[f"a{i}_obs"] = x
        out[f"a{i}_logits"] = logits.numpy()
        out[f"a{i}_value"] = value.numpy()
    np.savez_compressed(os.path.join(OUT, "policy.npz"), **out)


if __name__ == "__main__":
    main()
