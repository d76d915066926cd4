"""Env sharding across GPUs (one process per GPU) and the episode-stats reduce.

Environments never interact, so a batch of ``global_n`` envs is
split into contiguous shards; shard ``r`` owns global env indices
``[offset, offset + n)`` and seeds env ``i`` from
``SeedSequence(seed).spawn(...)[offset + i]`` (reference spawn_rngs,
env.py:591-594). Every per-env output is therefore bit-identical for any
number of GPUs. The only collective is a sum of five float64 episode counters
(count, reward, length, start loss, final loss) accumulated on device by the
step kernel -- one ``all_reduce`` every K steps, off the critical path.
"""
from __future__ import annotations

from dataclasses import dataclass

STAT_NAMES = ("episodes", "episode_reward", "episode_length", "episode_start_loss", "final_loss")


def shard(global_n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split: returns (global offset, count) of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if global_n < world:
        raise ValueError("fewer environments than ranks")
    base, extra = divmod(global_n, world)
    n = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, n


@dataclass
class EpisodeSummary:
    episodes: float
    mean_reward: float
    mean_length: float
    mean_start_loss: float
    mean_final_loss: float


class EpisodeStats:
    """float64[5] accumulator (device resident; the step kernel adds to it)."""

    def __init__(self, device="cpu"):
        import torch
        self.t = torch.zeros(5, dtype=torch.float64, device=device)

    def add_info(self, info) -> None:
        """Host-side accumulation from a step's info dict (used where the
        kernel accumulator is not in play, e.g. CPU tests)."""
        import torch
        done = torch.as_tensor(info["terminal"]).to(self.t.device).bool()
        vals = [done.double().sum()]
        for k in STAT_NAMES[1:]:
            vals.append(torch.as_tensor(info[k]).to(self.t.device).double()[done].sum())
        self.t += torch.stack(vals)

    def all_reduce(self, group=None):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(self.t, op=dist.ReduceOp.SUM, group=group)
        return self.t

    def summary(self) -> EpisodeSummary:
        v = [float(x) for x in self.t.cpu()]
        n = max(v[0], 1.0)
        return EpisodeSummary(v[0], v[1] / n, v[2] / n, v[3] / n, v[4] / n)


def max_over_ranks(value: float, device="cpu") -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])
