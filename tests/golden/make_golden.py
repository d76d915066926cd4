"""Generate the golden parity fixtures from the LIVE reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``levelgen`` from /root/reference/pkg/src, runs the reference's
own code on seeded inputs, and writes small ``.npz`` fixtures next to this
file. The fixtures are committed; nothing on the GPU box reads the reference.

Turtle and wide are not in the reference. Their fixtures
come from ``TurtleCore`` / ``WideCore`` below: subclasses of the reference's
own ``levelgen.env._Core`` that override only action application, position
and observation window; reset, metrics, loss,
reward, termination and auto-reset stay the reference's code.
"""
from __future__ import annotations

import hashlib
import itertools
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from levelgen import env as E  # noqa: E402
from levelgen import problems as P  # noqa: E402
from levelgen.tiles import get_domain  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------------------
# turtle / wide on top of the reference core
# ---------------------------------------------------------------------------


def wide_observation(core) -> np.ndarray:
    """Full-max-grid window: build_observation semantics with origin (0, 0)."""
    d = core.domain
    b, h, w = core.tiles.shape
    n_planes = d.n_tiles + 1
    planes = core.tiles[:, None, :, :] == np.arange(n_planes).reshape(1, n_planes, 1, 1)
    chans = [planes.astype(np.float32), core.frozen[:, None].astype(np.float32)]
    if core.control:
        cap = core.caps.astype(np.float64)
        ctrl = np.empty((b, len(core.control)), dtype=np.float64)
        for k, m in enumerate(core.control):
            target = (core.lo[m].astype(np.float64) + core.hi[m].astype(np.float64)) / 2.0
            ctrl[:, k] = (core.values[m].astype(np.float64) - target) / cap
        chans.append(np.broadcast_to(ctrl.astype(np.float32)[:, :, None, None],
                                     (b, len(core.control), h, w)).copy())
    return np.concatenate(chans, axis=1)


class _RepCore(E._Core):
    rep = "narrow"

    def n_actions(self) -> int:
        n = self.domain.n_tiles
        return 4 + n if self.rep == "turtle" else self.h * self.w * n

    def _apply(self, actions):
        raise NotImplementedError

    def step(self, actions, *, auto_reset):
        cfg = self.cfg
        actions = np.asarray(actions, dtype=np.int64)
        if actions.shape != (self.b,):
            raise ValueError("bad shape")
        if np.any((actions < 0) | (actions >= self.n_actions())):
            raise ValueError("action id out of range")
        rows = np.arange(self.b)
        wrote, r, c, tile = self._apply(actions)
        reward = np.zeros(self.b, dtype=np.float64)
        if wrote.any():
            hot = np.flatnonzero(wrote)
            self.tiles[hot, r[hot], c[hot]] = tile[hot].astype(np.uint8)
            self.changes[hot] += 1
            before = self.prev_loss[hot].copy()
            after = self._recompute(hot, reset=False)
            reward[hot] = before - after
        self.ep_reward += reward
        self.t += 1
        done = self.t >= self.max_steps
        if cfg.change_budget is not None:
            done |= self.changes >= cfg.change_budget
        info = {
            "terminal": done.copy(),
            "episode_reward": np.where(done, self.ep_reward, 0.0),
            "episode_length": np.where(done, self.t, 0),
            "episode_start_loss": np.where(done, self.ep_start_loss, 0.0),
            "final_loss": np.where(done, self.prev_loss, 0.0),
        }
        del rows
        if auto_reset and done.any():
            self.reset_rows(np.flatnonzero(done))
        return reward, done, info


class TurtleCore(_RepCore):
    rep = "turtle"

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.pos = np.zeros((self.b, 2), dtype=np.int64)

    def reset_rows(self, idx):
        super().reset_rows(idx)
        idx = np.asarray(idx, dtype=np.int64)
        first = self.order[idx, 0].astype(np.int64)
        self.pos[idx, 0], self.pos[idx, 1] = np.divmod(first, self.w)

    def positions(self):
        return self.pos.copy()

    def _apply(self, actions):
        n = self.domain.n_tiles
        r, c = self.pos[:, 0].copy(), self.pos[:, 1].copy()
        h, w = self.shape_hw[:, 0], self.shape_hw[:, 1]
        move = actions < 4
        r = np.where(move & (actions == 0), np.maximum(r - 1, 0), r)
        r = np.where(move & (actions == 1), np.minimum(r + 1, h - 1), r)
        c = np.where(move & (actions == 2), np.maximum(c - 1, 0), c)
        c = np.where(move & (actions == 3), np.minimum(c + 1, w - 1), c)
        self.pos[:, 0], self.pos[:, 1] = r, c
        rows = np.arange(self.b)
        tile = np.where(move, 0, actions - 4)
        editable = self.active[rows, r, c] & ~self.frozen[rows, r, c]
        cur = self.tiles[rows, r, c].astype(np.int64)
        wrote = ~move & editable & (tile != cur)
        del n
        return wrote, r, c, tile


class WideCore(_RepCore):
    rep = "wide"

    def _apply(self, actions):
        n = self.domain.n_tiles
        cell, tile = np.divmod(actions, n)
        r, c = np.divmod(cell, self.w)
        rows = np.arange(self.b)
        editable = self.active[rows, r, c] & ~self.frozen[rows, r, c]
        cur = self.tiles[rows, r, c].astype(np.int64)
        wrote = editable & (tile != cur)
        return wrote, r, c, tile

    def observe(self):
        return wide_observation(self)


class RefEnv:
    """BatchEnv-equivalent driver over a (possibly subclassed) reference core."""

    def __init__(self, cfg, n, seed, rep="narrow"):
        core_cls = {"narrow": E._Core, "turtle": TurtleCore, "wide": WideCore}[rep]
        self.core = core_cls(cfg, n, E.spawn_rngs(seed, n))
        self.rep = rep
        self.n_actions = cfg.n_actions if rep == "narrow" else self.core.n_actions()

    def reset(self):
        self.core.reset_rows(np.arange(self.core.b))
        return self.core.observe()

    def step(self, a):
        reward, done, info = self.core.step(a, auto_reset=True)
        return self.core.observe(), reward, done, info


# ---------------------------------------------------------------------------
# fixtures
# ---------------------------------------------------------------------------

ENV_CASES = {
    # name: (EnvConfig kwargs, representation, n_envs, steps)
    "c1_binary16_narrow_o31": (dict(domain="binary"), "narrow", 64, 800),
    "maze16_narrow_o31": (dict(domain="maze"), "narrow", 64, 200),
    "dungeon16_narrow_pins_rand": (dict(domain="dungeon", pinpoints=("player", "key", "door"),
                                        randomize_shape=True), "narrow", 64, 200),
    "binary64_narrow_o7": (dict(domain="binary", max_width=64, max_height=64, obs_size=7),
                           "narrow", 24, 120),
    "binary_ctrl_det_budget": (dict(domain="binary", max_width=7, max_height=9, obs_size=6,
                                    randomize_shape=True, deterministic_metrics=True,
                                    controllable=("diameter", "regions"), change_budget=12,
                                    init_weights={"air": 0.7, "wall": 0.3}), "narrow", 48, 300),
    "maze_ctrl_weights": (dict(domain="maze", max_width=8, max_height=5, obs_size=4,
                               controllable=("path_length",), pinpoints=("player", "door"),
                               loss_weights={"regions": 0.25, "path_length": 2.0},
                               max_steps=50), "narrow", 48, 300),
    "dungeon6_c5_like": (dict(domain="dungeon", max_width=6, max_height=6, obs_size=5,
                              randomize_shape=True, pinpoints=("player", "key", "door"),
                              max_steps=40, change_budget=10,
                              controllable=("pkd_path", "n_enemy")), "narrow", 48, 300),
    "maze_weighted_init": (dict(domain="maze", max_width=12, max_height=10, obs_size=9,
                                init_mode="weighted", randomize_shape=True), "narrow", 32, 200),
    "dungeon_weighted_init_o8": (dict(domain="dungeon", max_width=10, max_height=12, obs_size=8,
                                      init_mode="weighted",
                                      init_weights={"air": 5.0, "wall": 2.0, "enemy": 0.5,
                                                    "key": 0.3, "door": 0.3, "player": 0.3}),
                                 "narrow", 32, 200),
    "binary32x20_o15": (dict(domain="binary", max_width=20, max_height=32, obs_size=15),
                        "narrow", 32, 200),
    "binary48x40_o31_rand": (dict(domain="binary", max_width=40, max_height=48, obs_size=31,
                                  randomize_shape=True), "narrow", 16, 150),
    "c2_maze16_turtle_o31": (dict(domain="maze"), "turtle", 64, 300),
    "turtle_dungeon_pins": (dict(domain="dungeon", max_width=8, max_height=8, obs_size=7,
                                 pinpoints=("player", "key", "door"), randomize_shape=True,
                                 max_steps=60, controllable=("nearest_enemy",)),
                            "turtle", 48, 300),
    "c3_dungeon16_wide_pins_rand": (dict(domain="dungeon", pinpoints=("player", "key", "door"),
                                         randomize_shape=True), "wide", 64, 200),
    "wide_binary_ctrl": (dict(domain="binary", max_width=9, max_height=7, randomize_shape=True,
                              controllable=("regions",), change_budget=15), "wide", 48, 300),
}


def env_case(name, kw, rep, n, steps, seed=0):
    cfg = E.EnvConfig(**kw)
    env = RefEnv(cfg, n, seed, rep)
    act = np.random.default_rng(n)
    obs = env.reset()
    core = env.core
    d = core.domain
    reset_state = {
        "tiles": core.tiles.copy(), "frozen": core.frozen.copy(),
        "values": np.stack([core.values[m] for m in d.metric_names]),
        "unreach": np.stack([core.unreach[m] for m in d.metric_names]),
        "prev_loss": core.prev_loss.copy(),
    }
    actions = np.zeros((steps, n), dtype=np.int64)
    rewards = np.zeros((steps, n), dtype=np.float64)
    dones = np.zeros((steps, n), dtype=bool)
    info_keys = ("episode_reward", "episode_length", "episode_start_loss", "final_loss")
    infos = {k: np.zeros((steps, n), dtype=np.float64 if k != "episode_length" else np.int64)
             for k in info_keys}
    obs_digests = [digest(obs)]
    for t in range(steps):
        a = act.integers(0, env.n_actions, size=n)
        actions[t] = a
        obs, r, dn, info = env.step(a)
        rewards[t], dones[t] = r, dn
        for k in info_keys:
            infos[k][t] = info[k]
        obs_digests.append(digest(obs))
    rng = np.array([[st["state"]["state"] >> 64, st["state"]["state"] & ((1 << 64) - 1),
                     st["state"]["inc"] >> 64, st["state"]["inc"] & ((1 << 64) - 1),
                     st["has_uint32"], st["uinteger"]]
                    for st in (g.bit_generator.state for g in core.rngs)], dtype=np.uint64)
    pos = core.positions() if rep != "wide" else np.zeros((n, 2), dtype=np.int64)
    out = dict(
        config=np.array(repr(kw)), representation=np.array(rep), n_envs=n, steps=steps, seed=seed,
        actions=actions, rewards=rewards, dones=dones,
        obs_digests=np.array(obs_digests), final_obs=obs if obs.nbytes <= (2 << 20) else np.zeros(0),
        final_tiles=core.tiles.copy(), final_frozen=core.frozen.copy(),
        final_values=np.stack([core.values[m] for m in d.metric_names]),
        final_unreach=np.stack([core.unreach[m] for m in d.metric_names]),
        final_pos_idx=core.pos_idx.copy(), final_pos=pos, final_t=core.t.copy(),
        final_changes=core.changes.copy(), final_prev_loss=core.prev_loss.copy(),
        final_ep_reward=core.ep_reward.copy(), final_shape_hw=core.shape_hw.copy(),
        final_rng=rng, final_metric_seeds=core.metric_seeds.copy(),
        **{f"reset_{k}": v for k, v in reset_state.items()},
        **{f"info_{k}": v for k, v in infos.items()},
    )
    np.savez_compressed(os.path.join(OUT, f"env_{name}.npz"), **out)
    print(f"{name}: rewards sum {rewards.sum()} dones {dones.sum()}")


def metrics_fixture():
    """compute_metrics_batch on random maps, random active shapes, 3 domains."""
    rng = np.random.default_rng(2024)
    out = {}
    for domain in ("binary", "maze", "dungeon"):
        d = get_domain(domain)
        for (H, W, count) in ((3, 3, 200), (8, 8, 300), (16, 16, 600), (5, 13, 200),
                              (32, 32, 100), (64, 64, 60), (17, 50, 60)):
            tiles = np.full((count, H, W), d.border_id, dtype=np.uint8)
            active = np.zeros((count, H, W), dtype=bool)
            for i in range(count):
                h = int(rng.integers(1, H + 1)) if i % 2 else H
                w = int(rng.integers(1, W + 1)) if i % 2 else W
                if d.n_tiles == 2:
                    p = rng.uniform(0.2, 0.8)
                    g = (rng.random((h, w)) > p).astype(np.uint8)
                else:
                    probs = np.array([0.55, 0.25] + [0.2 / (d.n_tiles - 2)] * (d.n_tiles - 2))
                    g = rng.choice(d.n_tiles, size=(h, w), p=probs).astype(np.uint8)
                tiles[i, :h, :w] = g
                active[i, :h, :w] = True
            seeds = E.spawn_rngs(H * 1000 + W, count)
            vals, flags = P.compute_metrics_batch(d, tiles, active, seeds)
            key = f"{domain}_{H}x{W}"
            out[f"{key}_tiles"] = tiles
            out[f"{key}_active"] = active
            out[f"{key}_seed"] = np.array(H * 1000 + W)
            out[f"{key}_values"] = np.stack([vals[m] for m in d.metric_names])
            out[f"{key}_unreach"] = np.stack([flags[m] for m in d.metric_names])
    # exhaustive 3x3 binary (test_pathfind.py:32-50 style)
    maps = np.array(list(itertools.product([0, 1], repeat=9)), dtype=np.uint8).reshape(512, 3, 3)
    d = get_domain("binary")
    tiles = (1 - maps).astype(np.uint8)  # 1 = air -> tile 0
    active = np.ones_like(maps, dtype=bool)
    vals, flags = P.compute_metrics_batch(d, tiles, active, E.spawn_rngs(3, 512))
    out["exh3_tiles"] = tiles
    out["exh3_values"] = np.stack([vals[m] for m in d.metric_names])
    np.savez_compressed(os.path.join(OUT, "metrics.npz"), **out)
    print("metrics fixture written")


def rng_fixture():
    """Spawned PCG64 states and draw sequences as numpy produces them."""
    out = {}
    for seed in (0, 7, 123456789, 2 ** 40 + 3):
        ss = np.random.SeedSequence(seed)
        idx = np.array([0, 1, 2, 3, 100, 65535, 65536, 1048575], dtype=np.int64)
        kids = ss.spawn(int(idx.max()) + 1)
        states = []
        for i in idx:
            st = np.random.default_rng(kids[int(i)]).bit_generator.state
            s, inc = st["state"]["state"], st["state"]["inc"]
            states.append([s >> 64, s & ((1 << 64) - 1), inc >> 64, inc & ((1 << 64) - 1)])
        out[f"spawn_{seed}_idx"] = idx
        out[f"spawn_{seed}_states"] = np.array(states, dtype=np.uint64)
        g = np.random.default_rng(seed)
        st = g.bit_generator.state
        out[f"plain_{seed}_state"] = np.array(
            [st["state"]["state"] >> 64, st["state"]["state"] & ((1 << 64) - 1),
             st["state"]["inc"] >> 64, st["state"]["inc"] & ((1 << 64) - 1)], dtype=np.uint64)
        seq = []
        for k in range(400):
            seq.append(int(g.integers(0, [1, 2, 3, 7, 100, 257, 4097, 2 ** 31 + 5][k % 8])))
            seq.append(int(g.integers(0, 2 ** 63)))
            seq.append(int(np.float64(g.random()).view(np.uint64)))
        out[f"draws_{seed}"] = np.array(seq, dtype=np.uint64)
        ch = []
        for k in range(100):
            pop = 9 + 37 * k
            ch.extend(int(x) for x in g.choice(pop, size=1 + k % 5, replace=False))
        out[f"choice_{seed}"] = np.array(ch, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **out)
    print("rng fixture written")


if __name__ == "__main__":
    rng_fixture()
    metrics_fixture()
    for name, (kw, rep, n, steps) in ENV_CASES.items():
        env_case(name, kw, rep, n, steps)
