"""World-size-2 gloo tests of the env sharding and the episode-stats reduce (CPU).

Each rank steps its shard with the CPU oracle (the GPU kernels are pinned to
the same oracle by the gpu tests), so this checks the host-side partitioning
contract: shard offsets, per-env stream selection by global index, the stats
all-reduce and max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_12525_b200.config import EnvConfig
from paper_2408_12525_b200.sharding import EpisodeStats, max_over_ranks, shard

CFG = dict(domain="dungeon", max_width=6, max_height=6, obs_size=5, randomize_shape=True,
           pinpoints=("player", "key", "door"), max_steps=25, change_budget=8)
GLOBAL_N, STEPS, SEED = 37, 60, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        cfg = EnvConfig(**CFG)
        off, n = shard(GLOBAL_N, world, rank)
        env = O.OracleBatchEnv(cfg, n, seed=SEED, offset=off)
        env.reset()
        acts = np.random.default_rng(1).integers(0, cfg.n_actions, size=(STEPS, GLOBAL_N))
        stats = EpisodeStats("cpu")
        rewards = []
        for t in range(STEPS):
            obs, r, d, info = env.step(acts[t, off:off + n])
            stats.add_info(info)
            rewards.append(r)
        local = torch.from_numpy(np.stack(rewards, axis=1).copy())  # [n, STEPS]
        sizes = [shard(GLOBAL_N, world, k)[1] for k in range(world)]
        gathered = [torch.zeros((s, STEPS), dtype=torch.float64) for s in sizes]
        dist.all_gather(gathered, local) if len(set(sizes)) == 1 else _gather_ragged(gathered, local, rank)
        stats.all_reduce()
        slow = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((torch.cat(gathered).numpy(), stats.t.numpy().copy(), slow,
                   obs_digest(obs)))
    finally:
        dist.destroy_process_group()


def _gather_ragged(out, local, rank):
    for k, buf in enumerate(out):
        if k == rank:
            buf.copy_(local)
        dist.broadcast(buf, src=k)


def obs_digest(obs):
    return float(np.asarray(obs, dtype=np.float64).sum())


def test_shard_ranges_cover_batch():
    for n, w in ((10, 3), (1 << 20, 8), (37, 2), (8, 8)):
        spans = [shard(n, w, r) for r in range(w)]
        assert spans[0][0] == 0
        assert sum(c for _, c in spans) == n
        for (o1, c1), (o2, _) in zip(spans, spans[1:]):
            assert o1 + c1 == o2
    with pytest.raises(ValueError):
        shard(3, 4, 0)


def test_two_rank_gloo_sharding_matches_unsharded():
    from oracle import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rewards, stats, slow, _ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert slow == 2.0
    # unsharded reference run
    cfg = EnvConfig(**CFG)
    env = O.OracleBatchEnv(cfg, GLOBAL_N, seed=SEED)
    env.reset()
    acts = np.random.default_rng(1).integers(0, cfg.n_actions, size=(STEPS, GLOBAL_N))
    ref = EpisodeStats("cpu")
    rr = []
    for t in range(STEPS):
        _, r, _, info = env.step(acts[t])
        ref.add_info(info)
        rr.append(r)
    assert np.array_equal(rewards, np.stack(rr, axis=1))
    assert np.allclose(stats, ref.t.numpy(), rtol=1e-12, atol=0)
    assert stats[0] > 0  # episodes finished and were counted
