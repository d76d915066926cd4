"""Policy consumer of the observation on the GPU.

The reference feeds ``BatchEnv`` observations to a conv actor-critic
(``levelgen/nets.py:150-183``) inside ``ppo.collect_rollout``
(``levelgen/ppo.py:101-143``). This module keeps that consumer on the device:

* ``ArchConfig`` / ``ConvPolicy`` mirror ``nets.ArchConfig`` / ``nets.ConvPolicy``
  with the same module layout and parameter names (``trunk.<i>``,
  ``policy_head``, ``value_head``), so ``state_dict``s move between the two;
* ``conv1_bits`` runs the trunk's first layer (``Conv2d(C, K, 3)`` + ReLU)
  straight from the packed observation stream of a ``BatchEnv(obs_dtype="bits")``
  with the ``lg_conv1_bits`` CUDA kernel: 1 bit per input element is read
  instead of a float32, and the float32 observation is never written;
* ``PackedPolicy`` = that first layer + the rest of the trunk and the heads
  in torch (cuDNN/cuBLAS), numerically the same function as
  ``ConvPolicy(unpack(bits))`` up to float32 summation order;
* ``collect_rollout`` mirrors ``ppo.collect_rollout`` on device tensors.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class ArchConfig:
    """nets.ArchConfig (nets.py:33-70): widths of the conv trunk and FC stack."""
    obs_size: int
    in_channels: int
    n_actions: int
    conv_channels: tuple = (16, 32)
    fc_dims: tuple = (64,)

    def __post_init__(self) -> None:
        if self.obs_size < 1 or self.in_channels < 1:
            raise ValueError("bad observation dimensions")
        if self.n_actions < 2:
            raise ValueError("need at least a no-op and one tile action")
        if not self.fc_dims:
            raise ValueError("at least one fully connected layer is required")
        if any(c < 1 for c in self.conv_channels) or any(d < 1 for d in self.fc_dims):
            raise ValueError("layer widths must be positive")
        if self.conv_side() < 1:
            raise ValueError(f"{len(self.conv_channels)} 3x3 valid convs need obs_size >= "
                             f"{2 * len(self.conv_channels) + 1}, got {self.obs_size}")

    def conv_side(self) -> int:
        return self.obs_size - 2 * len(self.conv_channels)

    def flat_dim(self) -> int:
        c = self.conv_channels[-1] if self.conv_channels else self.in_channels
        return c * self.conv_side() ** 2


def default_arch(obs_size: int, in_channels: int, n_actions: int) -> ArchConfig:
    """nets.default_arch (nets.py:73-82)."""
    return ArchConfig(obs_size, in_channels, n_actions, (16, 32) if obs_size >= 5 else (16,), (64,))


def count_params(arch: ArchConfig) -> int:
    """nets.count_params (nets.py:85-98)."""
    n, cin = 0, arch.in_channels
    for cout in arch.conv_channels:
        n += 9 * cin * cout + cout
        cin = cout
    d = arch.flat_dim()
    for h in arch.fc_dims:
        n += d * h + h
        d = h
    return n + d * arch.n_actions + arch.n_actions + d + 1


def _torch():
    import torch
    return torch


def make_policy(arch: ArchConfig):
    """nets.ConvPolicy (nets.py:150-183): conv trunk (3x3 valid + ReLU each),
    flatten, FC stack with ReLU, linear policy and value heads. Orthogonal
    init (gain sqrt 2; heads 0.01 and 1.0), zero biases, as nets.layer_init."""
    torch = _torch()
    nn = torch.nn

    def init(layer, gain=float(np.sqrt(2))):
        nn.init.orthogonal_(layer.weight, gain)
        nn.init.constant_(layer.bias, 0.0)
        return layer

    class ConvPolicy(nn.Module):
        def __init__(self):
            super().__init__()
            self.arch = arch
            mods, cin = [], arch.in_channels
            for cout in arch.conv_channels:
                mods += [init(nn.Conv2d(cin, cout, kernel_size=3)), nn.ReLU()]
                cin = cout
            mods.append(nn.Flatten())
            d = arch.flat_dim()
            for h in arch.fc_dims:
                mods += [init(nn.Linear(d, h)), nn.ReLU()]
                d = h
            self.trunk = nn.Sequential(*mods)
            self.policy_head = init(nn.Linear(d, arch.n_actions), 0.01)
            self.value_head = init(nn.Linear(d, 1), 1.0)

        def forward(self, obs):
            want = (arch.in_channels, arch.obs_size, arch.obs_size)
            if obs.ndim != 4 or tuple(obs.shape[1:]) != want:
                raise ValueError(f"expected [batch, {want[0]}, {want[1]}, {want[2]}] observations, "
                                 f"got {tuple(obs.shape)}")
            h = self.trunk(obs)
            return self.policy_head(h), self.value_head(h).squeeze(-1)

    return ConvPolicy()


def init_policy(arch: ArchConfig, seed: int):
    """nets.init_policy (nets.py:186-189): same seed, same weights."""
    _torch().manual_seed(seed)
    return make_policy(arch)


CHECKPOINT_FORMAT = "levelgen-checkpoint"
CHECKPOINT_VERSION = 1


@dataclass
class Checkpoint:
    """nets.Checkpoint (nets.py:204-239): ``meta`` JSON + named arrays, the
    reference's on-disk ``.npz`` format (``param/<name>`` = model weights)."""
    meta: dict
    arrays: dict

    @property
    def arch(self) -> ArchConfig:
        a = self.meta["arch"]
        return ArchConfig(obs_size=a["obs_size"], in_channels=a["in_channels"], n_actions=a["n_actions"],
                          conv_channels=tuple(a["conv_channels"]), fc_dims=tuple(a["fc_dims"]))

    @property
    def step(self) -> int:
        return int(self.meta["step"])

    def build_model(self, device=None):
        torch = _torch()
        model = make_policy(self.arch)
        state = {k[len("param/"):]: torch.from_numpy(np.array(v, dtype=np.float32))
                 for k, v in self.arrays.items() if k.startswith("param/")}
        model.load_state_dict(state)
        return model.to(device) if device is not None else model


def save_checkpoint(path, model, *, env_config: dict, step: int, extra_meta: dict | None = None) -> str:
    """nets.save_checkpoint (nets.py:242-270): little-endian float32 params."""
    import json
    from dataclasses import asdict
    meta = {"format": CHECKPOINT_FORMAT, "version": CHECKPOINT_VERSION, "arch": asdict(model.arch),
            "env": env_config, "step": int(step)}
    if extra_meta:
        meta.update(extra_meta)
    arrays = {f"param/{k}": v.detach().cpu().numpy().astype("<f4") for k, v in model.state_dict().items()}
    with open(path, "wb") as f:
        np.savez(f, meta=np.array(json.dumps(meta)), **arrays)
    return str(path)


def load_checkpoint(path) -> Checkpoint:
    """nets.load_checkpoint (nets.py:273-282), same format checks and errors."""
    import json
    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(str(z["meta"]))
        if meta.get("format") != CHECKPOINT_FORMAT:
            raise ValueError(f"{path}: not a recognized checkpoint")
        if meta.get("version") != CHECKPOINT_VERSION:
            raise ValueError(f"{path}: unsupported checkpoint version {meta.get('version')}")
        arrays = {k: z[k] for k in z.files if k != "meta"}
    return Checkpoint(meta=meta, arrays=arrays)


def conv1_bits(bits, n_envs: int, obs_shape, weight, bias, *, out_dtype=None, relu: bool = True, out=None,
               channels_last: bool = False):
    """relu(conv2d(obs, weight, bias)) (3x3, valid) from the packed stream of a
    ``BatchEnv(obs_dtype="bits")``; obs_shape = (C, OH, OW). Output
    [n_envs, K, OH-2, OW-2] in float32 (default) or bfloat16; with
    ``channels_last`` the same logical tensor in torch's channels-last layout
    (the kernel then writes each pixel's K channels with vector stores)."""
    torch = _torch()
    C, OH, OW = (int(x) for x in obs_shape)
    K = int(weight.shape[0])
    if tuple(weight.shape) != (K, C, 3, 3):
        raise ValueError(f"weight must be [K, {C}, 3, 3], got {tuple(weight.shape)}")
    out_dtype = out_dtype or torch.float32
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out_dtype must be float32 or bfloat16")
    w = weight.detach().to(torch.float32).contiguous()
    b = bias.detach().to(torch.float32).contiguous()
    if out is None:
        if channels_last:
            out = torch.empty((n_envs, OH - 2, OW - 2, K), dtype=out_dtype, device=bits.device).permute(0, 3, 1, 2)
        else:
            out = torch.empty((n_envs, K, OH - 2, OW - 2), dtype=out_dtype, device=bits.device)
    nhwc = int(out.dim() == 4 and out.stride(1) == 1 and K > 1)
    stream = ctypes.c_void_p(torch.cuda.current_stream(bits.device).cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.load().lg_conv1_bits(p(bits), int(n_envs), C, OH, OW, p(w), p(b), K, p(out),
                                         int(out_dtype == torch.bfloat16), int(relu), nhwc, stream))
    return out


class PackedPolicy:
    """A ConvPolicy evaluated from packed observation bits: the first conv +
    ReLU by ``lg_conv1_bits``, the rest of the trunk and both heads by the
    model's own torch modules (optionally under bf16 autocast)."""

    def __init__(self, model, obs_shape, *, bf16: bool = False, channels_last: bool = False):
        if not model.arch.conv_channels:
            raise ValueError("the packed path needs at least one conv layer")
        self.model = model
        self.obs_shape = tuple(obs_shape)
        self.bf16 = bf16
        self.channels_last = channels_last
        if channels_last:  # the rest of the conv trunk in NHWC: converts the model's conv weights in place
            torch = _torch()
            for m in model.trunk:
                if isinstance(m, torch.nn.Conv2d):
                    m.to(memory_format=torch.channels_last)
        self.conv1 = model.trunk[0]
        self.rest = model.trunk[2:]  # after Conv2d + ReLU

    def __call__(self, bits, n_envs: int):
        torch = _torch()
        h = conv1_bits(bits, n_envs, self.obs_shape, self.conv1.weight, self.conv1.bias,
                       out_dtype=torch.bfloat16 if self.bf16 else torch.float32,
                       channels_last=self.channels_last)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.bf16):
            h = self.rest(h)
            return self.model.policy_head(h).float(), self.model.value_head(h).squeeze(-1).float()


def pack_conv2_weight(weight):
    """Conv2d(16 -> 32, 3x3) weight [32, 16, 3, 3] -> the trunk kernel's B
    operands: per kernel row dy an N = 96 x K = 16 bf16 block of UMMA K-major
    core matrices whose rows are the 32 output channels of taps (dy, 2),
    (dy, 1), (dy, 0) in that order, [3, 1536] (csrc/trunk_kernel.cuh)."""
    torch = _torch()
    n, k = weight.shape[:2]
    w = weight.detach().to(torch.float32).flip(3).permute(2, 3, 0, 1)  # [dy][2 - dx][n][k]
    w = w.reshape(3, 3 * n // 8, 8, k // 8, 8)
    return w.permute(0, 3, 1, 2, 4).reshape(3, 3 * n * k).to(torch.bfloat16).contiguous()


def pack_fc_weight(weight, channels: int, side: int):
    """Linear(channels * side^2 -> 64) weight [64, channels*side^2] (torch
    flattens [C, H, W]) -> per conv2 pixel an N = 64 x K = channels bf16
    block of UMMA K-major core matrices, [side^2, 64 * channels]."""
    torch = _torch()
    nout = weight.shape[0]
    npx = side * side
    w = weight.detach().to(torch.float32).reshape(nout, channels, npx).permute(2, 0, 1)  # [p][n][k]
    w = w.reshape(npx, nout // 8, 8, channels // 8, 8).permute(0, 3, 1, 2, 4)
    return w.reshape(npx, nout * channels).to(torch.bfloat16).contiguous()


class TrunkPolicy:
    """The default ConvPolicy (conv (16, 32), fc (64,); nets.py:150-183)
    evaluated from packed observation bits on the GPU with two kernels and no
    torch math: ``lg_conv1_bits`` writes relu(conv1) as bf16 tensor-core tiles,
    ``lg_policy_trunk`` runs conv2 + ReLU, the FC + ReLU (tcgen05.mma, TMEM
    accumulators) and both heads (fp32). bf16 operands, fp32 accumulation.
    Call ``refresh()`` after the model's weights change (an optimizer step)."""

    def __init__(self, model, obs_shape):
        arch = model.arch
        if tuple(arch.conv_channels) != (16, 32) or tuple(arch.fc_dims) != (64,):
            raise ValueError("the fused trunk implements the default arch: conv (16, 32), fc (64,)")
        if arch.n_actions > 16:
            raise ValueError("the fused trunk's heads support at most 16 actions")
        C, OH, OW = (int(x) for x in obs_shape)
        if OH != OW or OH < 5:
            raise ValueError("the fused trunk needs a square window of side >= 5")
        self.model = model
        self.obs_shape = (C, OH, OW)
        self.P1 = OH - 2
        self.refresh()

    def refresh(self) -> None:
        torch = _torch()
        m = self.model
        conv1, conv2, fc = m.trunk[0], m.trunk[2], m.trunk[5]
        P2 = self.P1 - 2
        with torch.no_grad():
            self.w1 = conv1.weight.detach().float().contiguous()
            self.b1 = conv1.bias.detach().float().contiguous()
            self.w2 = pack_conv2_weight(conv2.weight)
            self.b2 = conv2.bias.detach().float().contiguous()
            self.w3 = pack_fc_weight(fc.weight, 32, P2)
            self.b3 = fc.bias.detach().float().contiguous()
            self.wh = torch.cat([m.policy_head.weight, m.value_head.weight]).detach().float().contiguous()
            self.bh = torch.cat([m.policy_head.bias, m.value_head.bias]).detach().float().contiguous()

    def conv1_tiles(self, bits, n_envs: int):
        torch = _torch()
        tiles = (n_envs + 127) // 128
        out = torch.empty(tiles * self.P1 * self.P1 * 2048, dtype=torch.bfloat16, device=bits.device)
        C, OH, OW = self.obs_shape
        stream = ctypes.c_void_p(torch.cuda.current_stream(bits.device).cuda_stream)
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.load().lg_conv1_bits(p(bits), int(n_envs), C, OH, OW, p(self.w1), p(self.b1), 16, p(out),
                                             1, 1, 2, stream))
        return out

    def __call__(self, bits, n_envs: int):
        torch = _torch()
        c1 = self.conv1_tiles(bits, n_envs)
        na = self.model.arch.n_actions
        logits = torch.empty((n_envs, na), dtype=torch.float32, device=bits.device)
        value = torch.empty(n_envs, dtype=torch.float32, device=bits.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(bits.device).cuda_stream)
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.load().lg_policy_trunk(p(c1), int(n_envs), self.P1, p(self.w2), p(self.b2), p(self.w3),
                                               p(self.b3), p(self.wh), p(self.bh), na, p(logits), p(value), stream))
        return logits, value

    def sample(self, bits, n_envs: int, seed: int, actions=None, logp=None, value=None):
        """The forward pass plus ppo.collect_rollout's action draw
        (ppo.py:125-130: Categorical(logits).sample(), log_prob) fused into the
        trunk kernel's heads: returns (actions int64, logp f32, value f32,
        logits f32). Env i's uniform is a counter hash of (seed, i)."""
        torch = _torch()
        c1 = self.conv1_tiles(bits, n_envs)
        na = self.model.arch.n_actions
        dev = bits.device
        logits = torch.empty((n_envs, na), dtype=torch.float32, device=dev)
        value = torch.empty(n_envs, dtype=torch.float32, device=dev) if value is None else value
        actions = torch.empty(n_envs, dtype=torch.int64, device=dev) if actions is None else actions
        logp = torch.empty(n_envs, dtype=torch.float32, device=dev) if logp is None else logp
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.load().lg_policy_trunk_sample(
            p(c1), int(n_envs), self.P1, p(self.w2), p(self.b2), p(self.w3), p(self.b3), p(self.wh), p(self.bh), na,
            p(logits), p(value), int(seed) & ((1 << 64) - 1), p(actions), p(logp), stream))
        return actions, logp, value, logits


@dataclass
class RolloutBatch:
    """ppo.RolloutBatch (ppo.py:91-98), device tensors; obs in the env's format."""
    obs: object       # [T, *obs] (float32 [T,B,C,O,O], or packed int32 [T, words])
    actions: object   # [T, B] int64
    logprobs: object  # [T, B] float32
    rewards: object   # [T, B] float64
    values: object    # [T, B] float32
    dones: object     # [T, B] bool


def collect_rollout(policy, env, length: int, sampler, obs):
    """ppo.collect_rollout (ppo.py:101-143) on the GPU: ``length`` lockstep
    steps sampling actions from ``policy`` (a ConvPolicy taking float32
    observations, or a PackedPolicy for an ``obs_dtype="bits"`` env). Returns
    the batch, the observation after the last step and the rewards of the
    episodes that finished (one host sync at the end, not one per step)."""
    torch = _torch()
    B = env.n_envs
    packed = isinstance(policy, (PackedPolicy, TrunkPolicy))
    dev = env.device
    out_obs = torch.empty((length,) + tuple(obs.shape), dtype=obs.dtype, device=dev)
    out_actions = torch.empty((length, B), dtype=torch.int64, device=dev)
    out_logprobs = torch.empty((length, B), dtype=torch.float32, device=dev)
    out_rewards = torch.empty((length, B), dtype=torch.float64, device=dev)
    out_values = torch.empty((length, B), dtype=torch.float32, device=dev)
    out_dones = torch.empty((length, B), dtype=torch.bool, device=dev)
    finished_sum = []
    fused = isinstance(policy, TrunkPolicy)
    if fused:  # the draw happens in the trunk kernel: per-step seeds from the sampler's seed, no sync
        base = sampler.initial_seed()
        policy._draws = getattr(policy, "_draws", 0)
    with torch.no_grad():
        for t in range(length):
            if fused:
                policy._draws += 1
                seed = (base * 0x9E3779B97F4A7C15 + policy._draws) & ((1 << 64) - 1)
                policy.sample(obs, B, seed, actions=out_actions[t], logp=out_logprobs[t], value=out_values[t])
                out_obs[t].copy_(obs)
                obs, reward, done, info = env.step(out_actions[t], checked=True)  # sampled: in range
                out_rewards[t] = reward
                out_dones[t] = done
                finished_sum.append(info["episode_reward"])
                continue
            logits, value = policy(obs, B) if packed else policy(obs)
            probs = torch.softmax(logits.float(), dim=-1)
            actions = torch.multinomial(probs, 1, generator=sampler).squeeze(1)
            logp = torch.log_softmax(logits.float(), dim=-1).gather(1, actions[:, None]).squeeze(1)
            out_obs[t].copy_(obs)
            out_actions[t] = actions
            out_logprobs[t] = logp
            out_values[t] = value.float()
            obs, reward, done, info = env.step(actions, checked=True)  # sampled: in range
            out_rewards[t] = reward
            out_dones[t] = done
            finished_sum.append(info["episode_reward"])
    ep = torch.stack(finished_sum)
    finished = ep[out_dones].tolist()  # time-major, env order within a step (ppo.py:141-142)
    return RolloutBatch(out_obs, out_actions, out_logprobs, out_rewards, out_values, out_dones), obs, finished


__all__ = ["ArchConfig", "default_arch", "count_params", "make_policy", "init_policy", "conv1_bits",
           "Checkpoint", "save_checkpoint", "load_checkpoint", "TrunkPolicy", "pack_conv2_weight", "pack_fc_weight",
           "PackedPolicy", "RolloutBatch", "collect_rollout"]
