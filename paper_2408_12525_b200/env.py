"""``BatchEnv`` on B200: the reference's batched env API over the CUDA library.

Host mirror of ``levelgen.env.BatchEnv`` (reference env.py:486-588): same
constructor, properties, ``reset``/``step``/``observe``/``state_dict``/
``load_state_dict`` and the same exceptions, backed by the C ABI in
include/pcgrl_b200.h. Per-env random streams are
``SeedSequence(seed).spawn(...)[global_offset + i]`` exactly as
``spawn_rngs`` (env.py:591-594), so results are bit-identical to the
reference for the same seed and actions, and independent of how a batch is
sharded over GPUs.

Outputs are CUDA tensors (obs float32 [B,C,OH,OW], reward float64 [B], done
bool [B], info dict of [B] tensors). ``NumpyBatchEnv`` returns numpy arrays
like the reference, copying through host buffers inside the library call.
"""
from __future__ import annotations

import ctypes
from typing import Any

import numpy as np

from . import _lib
from .config import EnvConfig
from .tiles import get_domain

INFO_KEYS = ("terminal", "episode_reward", "episode_length", "episode_start_loss", "final_loss")


OBS_FORMATS = {"float32": 0, "uint8": 1, "bits": 2}


def make_lg_config(cfg: EnvConfig, obs_dtype: str = "float32") -> _lib.LgConfig:
    d = cfg.domain_obj
    c = _lib.LgConfig()
    if obs_dtype not in OBS_FORMATS:
        raise ValueError(f"unknown obs_dtype {obs_dtype!r}; expected one of {sorted(OBS_FORMATS)}")
    c.obs_format = OBS_FORMATS[obs_dtype]
    c.domain = d.code
    c.representation = ("narrow", "turtle", "wide").index(cfg.representation)
    c.max_h, c.max_w = cfg.max_height, cfg.max_width
    c.obs_size = cfg.obs_size
    c.randomize_shape = int(bool(cfg.randomize_shape))
    c.init_weighted = int((cfg.init_mode or d.default_init_mode) == "weighted")
    for i, v in enumerate(cfg.init_cdf()):
        c.init_cdf[i] = float(v)
    pins = [d.tile_id(t) for t in cfg.pinpoints]
    if len(pins) > 16:
        raise ValueError("at most 16 pinpoints are supported on device")
    c.n_pins = len(pins)
    for i, t in enumerate(pins):
        c.pins[i] = t
    ctrl = [i for i, m in enumerate(d.metric_names) if m in cfg.controllable]
    c.n_ctrl = len(ctrl)
    for i, m in enumerate(ctrl):
        c.ctrl[i] = m
    if cfg.max_steps is not None and cfg.max_steps >= 2 ** 62:
        raise ValueError("max_steps too large")
    c.max_steps = int(cfg.max_steps or 0)
    c.change_budget = int(cfg.change_budget or 0)
    c.det_metrics = int(bool(cfg.deterministic_metrics))
    w = cfg.weights()
    for i, m in enumerate(d.metric_names):
        c.weights[i] = float(w[m])
    return c


def _stream(torch, device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class BatchEnv:
    """Lockstep batch of identical-config environments with auto-reset."""

    def __init__(self, config: EnvConfig, n_envs: int, seed: int = 0, *, device: Any = None,
                 global_offset: int = 0, validate: bool = True, obs_dtype: str = "float32"):
        """``obs_dtype="uint8"`` (opt-in, configs without control planes) writes
        the same 0/1 observation planes as bytes: 4x less HBM traffic for
        consumers on the GPU; ``"bits"`` writes them as one packed int32 stream
        (32x less; see ``unpack_obs`` and ``policy.conv1_bits``). The default
        float32 matches the reference."""
        import torch

        self._torch = torch
        if n_envs < 1:
            raise ValueError("need at least one environment")
        lib = _lib.load()
        self._cfg = config
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.validate = validate
        self._global_offset = int(global_offset)
        self._seed = check_seed(seed)
        handle = ctypes.c_void_p()
        cfgc = make_lg_config(config, obs_dtype)
        self.obs_dtype = obs_dtype
        _lib.check(lib.lg_create(ctypes.byref(cfgc), int(n_envs), int(global_offset),
                                 self._seed, self.device.index, ctypes.byref(handle)))
        self._h = handle
        desc = _lib.LgDesc()
        _lib.check(lib.lg_describe(self._h, ctypes.byref(desc)))
        self._desc = desc
        self._n = int(n_envs)
        self._started = False

    # -- properties (env.py:499-514) ----------------------------------------
    @property
    def config(self) -> EnvConfig:
        return self._cfg

    @property
    def n_envs(self) -> int:
        return self._n

    @property
    def n_actions(self) -> int:
        return self._cfg.n_actions

    @property
    def observation_shape(self) -> tuple[int, int, int]:
        return (self._desc.obs_c, self._desc.obs_h, self._desc.obs_w)

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().lg_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- buffers -------------------------------------------------------------
    def new_obs(self):
        t = self._torch
        if self.obs_dtype == "bits":  # one packed stream: element i = bit i % 32 of word i // 32
            n = self._n * int(np.prod(self.observation_shape))
            return t.empty((n + 31) // 32, dtype=t.int32, device=self.device)
        dt = t.uint8 if self.obs_dtype == "uint8" else t.float32
        return t.empty((self._n,) + self.observation_shape, dtype=dt, device=self.device)

    def _info_buffers(self):
        t, B, dev = self._torch, self._n, self.device
        return {
            "terminal": t.empty(B, dtype=t.bool, device=dev),
            "episode_reward": t.empty(B, dtype=t.float64, device=dev),
            "episode_length": t.empty(B, dtype=t.int64, device=dev),
            "episode_start_loss": t.empty(B, dtype=t.float64, device=dev),
            "final_loss": t.empty(B, dtype=t.float64, device=dev),
        }

    # -- API -------------------------------------------------------------------
    def reset(self, out=None):
        obs = self.new_obs() if out is None else out
        with self._torch.cuda.device(self.device):
            _lib.check(_lib.load().lg_reset(self._h, _ptr(obs), _stream(self._torch, self.device)))
        self._started = True
        if self.validate:
            self.check_errors()
        return obs

    def _actions(self, actions):
        """-> (device int64 actions, whether the range still needs the device check)."""
        t = self._torch
        if isinstance(actions, t.Tensor):
            a = actions
            if a.shape != (self._n,):
                raise ValueError(f"expected {self._n} actions, got shape {tuple(a.shape)}")
            if a.device != self.device or a.dtype != t.int64:
                a = a.to(device=self.device, dtype=t.int64)
            return a.contiguous(), True
        a = np.asarray(actions, dtype=np.int64)
        if a.shape != (self._n,):
            raise ValueError(f"expected {self._n} actions, got shape {a.shape}")
        if a.size and (a.min() < 0 or a.max() >= self.n_actions):
            raise ValueError("action id out of range")
        return t.from_numpy(np.ascontiguousarray(a)).to(self.device, non_blocking=False), False

    def step(self, actions, *, out=None, stats=None, with_obs: bool = True, checked: bool = False):
        """One transition (env.py:521-525): ``(obs, reward, done, info)``.

        With ``validate`` (the default), device actions are range-checked on
        the device before the step kernel runs -- a bad batch raises
        ``ValueError`` and leaves every env untouched, as env.py:358-361 --
        and the auto-reset error flags (pinpoint overflow, no editable cell;
        ``reset_rows``, env.py:315-316, grid.py:213-214) are read back: one
        4-byte device->host read per step. ``validate=False`` (throughput) or
        ``checked=True`` (the caller guarantees the range, e.g. actions
        sampled from the policy) skips it; flags then surface on
        ``check_errors()``."""
        if not self._started:
            raise RuntimeError("reset() the batch before stepping")
        t = self._torch
        a, device_check = self._actions(actions)
        validate = self.validate and not checked
        obs = (self.new_obs() if out is None else out) if with_obs else None
        reward = t.empty(self._n, dtype=t.float64, device=self.device)
        done = t.empty(self._n, dtype=t.bool, device=self.device)
        info = self._info_buffers()
        ci = _lib.LgInfo(*[_ptr(info[k]) for k in INFO_KEYS])
        flags = _lib.STEP_VALIDATE if (validate and device_check) else 0
        with t.cuda.device(self.device):
            _lib.check(_lib.load().lg_step_flags(
                self._h, _ptr(a), _ptr(obs) if obs is not None else None, _ptr(reward), _ptr(done),
                ctypes.byref(ci), _ptr(stats) if stats is not None else None, flags,
                _stream(t, self.device)))
        if validate:
            self.check_errors()
        return obs, reward, done, info

    def step_raw(self, actions, obs, reward, done, info=None, stats=None) -> None:
        """Allocation-free step into caller-owned device tensors (bench path)."""
        ci = None
        if info is not None:
            ci = ctypes.byref(_lib.LgInfo(*[_ptr(info[k]) if k in info else None for k in INFO_KEYS]))
        _lib.check(_lib.load().lg_step(
            self._h, _ptr(actions), _ptr(obs) if obs is not None else None, _ptr(reward), _ptr(done),
            ci, _ptr(stats) if stats is not None else None, _stream(self._torch, self.device)))

    def _check_out(self, name, t, dtype, numel):
        if t.device != self.device or t.dtype != dtype or not t.is_contiguous() or t.numel() != numel:
            raise ValueError(f"{name}: expected a contiguous {dtype} tensor of {numel} elements on {self.device}, "
                             f"got {t.dtype} {tuple(t.shape)} on {t.device}")

    def step_random(self, seed: int, obs, reward, done, info=None, stats=None, actions_out=None) -> None:
        """harness.bench_random_fps's loop body (harness.py:149-175) on device:
        uniform actions (the draw of ``random_actions(seed)``, recorded in
        ``actions_out``) and the step, in one call. Consecutive calls overlap
        launch to launch (include/pcgrl_b200.h lg_step_random)."""
        t, B = self._torch, self._n
        if not self._started:
            raise RuntimeError("reset() the batch before stepping")
        if obs is not None:
            n_el = B * int(np.prod(self.observation_shape))
            if self.obs_dtype == "bits":
                self._check_out("obs", obs, t.int32, (n_el + 31) // 32)
            else:
                self._check_out("obs", obs, t.uint8 if self.obs_dtype == "uint8" else t.float32, n_el)
        self._check_out("reward", reward, t.float64, B)
        self._check_out("done", done, t.bool, B)
        if actions_out is not None:
            self._check_out("actions_out", actions_out, t.int64, B)
        if stats is not None:
            self._check_out("stats", stats, t.float64, 5)
        ci = None
        if info is not None:
            ci = ctypes.byref(_lib.LgInfo(*[_ptr(info[k]) if k in info else None for k in INFO_KEYS]))
        _lib.check(_lib.load().lg_step_random(
            self._h, int(seed) & ((1 << 64) - 1), _ptr(actions_out) if actions_out is not None else None,
            _ptr(obs) if obs is not None else None, _ptr(reward), _ptr(done), ci,
            _ptr(stats) if stats is not None else None, _stream(self._torch, self.device)))

    def observe(self, out=None):
        obs = self.new_obs() if out is None else out
        with self._torch.cuda.device(self.device):
            _lib.check(_lib.load().lg_observe(self._h, _ptr(obs), _stream(self._torch, self.device)))
        return obs

    def random_actions(self, seed: int, out=None):
        t = self._torch
        a = t.empty(self._n, dtype=t.int64, device=self.device) if out is None else out
        _lib.check(_lib.load().lg_random_actions(self._h, _ptr(a), int(seed) & ((1 << 64) - 1),
                                                 _stream(t, self.device)))
        return a

    def errors(self) -> int:
        flags = ctypes.c_uint32(0)
        _lib.check(_lib.load().lg_errors(self._h, ctypes.byref(flags), _stream(self._torch, self.device)))
        return int(flags.value)

    def check_errors(self) -> None:
        f = self.errors()
        if f & _lib.FLAG_BAD_ACTION:
            raise ValueError("action id out of range")
        if f & _lib.FLAG_PINPOINTS:
            raise ValueError("pinpoints requested but not enough free cells")
        if f & _lib.FLAG_NO_EDITABLE:
            raise ValueError("no editable cells: every active cell is frozen")

    # -- checkpoint support (env.py:535-585) ----------------------------------
    def _state_tensors(self):
        t, B, dev = self._torch, self._n, self.device
        cfg = self._cfg
        H, W, M = cfg.max_height, cfg.max_width, len(cfg.domain_obj.metric_names)
        spec = {
            "tiles": ((B, H, W), t.uint8), "active": ((B, H, W), t.uint8),
            "frozen": ((B, H, W), t.uint8), "shape_hw": ((B, 2), t.int64),
            "order": ((B, H * W), t.int32), "order_len": ((B,), t.int64),
            "pos_idx": ((B,), t.int64), "pos": ((B, 2), t.int64), "t": ((B,), t.int64),
            "changes": ((B,), t.int64), "max_steps": ((B,), t.int64), "lo": ((M, B), t.int64),
            "hi": ((M, B), t.int64), "values": ((M, B), t.int64), "unreach": ((M, B), t.uint8),
            "prev_loss": ((B,), t.float64), "ep_reward": ((B,), t.float64),
            "ep_start_loss": ((B,), t.float64), "metric_seeds": ((B,), t.int64),
            "rng": ((B, 6), t.int64),
        }
        return {k: t.empty(s, dtype=d, device=dev) for k, (s, d) in spec.items()}

    def state_tensors(self) -> dict:
        """Device-side state_dict (CUDA tensors, same keys/layout)."""
        ts = self._state_tensors()
        st = _lib.LgState(*[_ptr(ts[k]) for k in _lib.STATE_FIELDS])
        with self._torch.cuda.device(self.device):
            _lib.check(_lib.load().lg_export_state(self._h, ctypes.byref(st),
                                                   _stream(self._torch, self.device)))
        return ts

    def state_dict(self) -> dict[str, Any]:
        ts = self.state_tensors()
        out = {k: v.cpu().numpy() for k, v in ts.items()}
        for k in ("active", "frozen", "unreach"):
            out[k] = out[k].astype(bool)
        rng = out.pop("rng").view(np.uint64)
        out["rng"] = rng
        out["rng_states"] = [_rng_state_dict(r) for r in rng]
        out["started"] = np.array([self._started])
        return out

    def load_state_dict(self, state: dict[str, Any]) -> None:
        t = self._torch
        cfg = self._cfg
        B, W = self._n, cfg.max_width
        host = {}
        for k in _lib.STATE_FIELDS:
            if k == "rng":
                if "rng" in state:
                    v = np.asarray(state["rng"], dtype=np.uint64)
                else:
                    v = np.stack([_rng_row(s) for s in state["rng_states"]])
                host[k] = v.view(np.int64)
                continue
            if k == "pos":
                if "pos" in state and cfg.representation == "turtle":
                    v = np.asarray(state["pos"], dtype=np.int64)
                else:
                    order = np.asarray(state["order"])
                    idx = np.asarray(state["pos_idx"], dtype=np.int64)
                    flat = order[np.arange(B), np.clip(idx, 0, order.shape[1] - 1)].astype(np.int64)
                    flat = np.maximum(flat, 0)
                    v = np.stack([flat // W, flat % W], axis=1)
                host[k] = v
                continue
            v = np.asarray(state[k])
            if v.dtype == bool:
                v = v.astype(np.uint8)
            host[k] = v
        ref = self._state_tensors()
        dev = {}
        for k, v in host.items():
            npdt = _NP_OF[ref[k].dtype]
            dev[k] = t.from_numpy(np.ascontiguousarray(v).astype(npdt)).to(self.device).reshape(
                ref[k].shape)
        st = _lib.LgState(*[_ptr(dev[k]) for k in _lib.STATE_FIELDS])
        with t.cuda.device(self.device):
            _lib.check(_lib.load().lg_import_state(self._h, ctypes.byref(st), _stream(t, self.device)))
            t.cuda.current_stream(self.device).synchronize()
        if "started" in state:
            self._started = bool(np.asarray(state["started"]).ravel()[0])
        else:
            self._started = True

    def snapshot(self, i: int):
        """``EnvState`` of env ``i`` (reference env.py:527-528)."""
        from .scalar import _state_from_row
        return _state_from_row(self._cfg, _row(self.state_dict(), i), done=False)

    def grid_view(self, i: int):
        """``TileGrid`` of env ``i`` (reference env.py:530-531)."""
        return self.snapshot(i).grid


def _row(sd: dict, i: int) -> dict:
    """Slice a batch state_dict down to env ``i`` (B = 1)."""
    out = {}
    for k, v in sd.items():
        if k == "rng_states":
            out[k] = [v[i]]
        elif k == "started":
            out[k] = v
        elif k in ("lo", "hi", "values", "unreach"):
            out[k] = v[:, i:i + 1]
        else:
            out[k] = v[i:i + 1]
    return out


def _np_of():
    import torch
    return {torch.uint8: np.uint8, torch.int32: np.int32, torch.int64: np.int64,
            torch.float64: np.float64, torch.float32: np.float32, torch.bool: np.bool_}


class _LazyNp(dict):
    def __missing__(self, key):
        self.update(_np_of())
        return dict.__getitem__(self, key)


_NP_OF = _LazyNp()


def _rng_state_dict(row) -> dict:
    row = [int(x) for x in row]
    return {"bit_generator": "PCG64", "state": {"state": (row[0] << 64) | row[1],
                                                "inc": (row[2] << 64) | row[3]},
            "has_uint32": row[4], "uinteger": row[5]}


def _rng_row(st: dict) -> np.ndarray:
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"])],
                    dtype=np.uint64)


def check_seed(seed) -> int:
    """``SeedSequence(seed)`` takes any non-negative int and raises on negative
    ones (env.py:591-594); the device streams take the 64-bit seeds, so larger
    ones are refused instead of silently masked."""
    s = int(seed)
    if s < 0:
        raise ValueError("seed must be a non-negative integer")
    if s >= 1 << 64:
        raise ValueError("seeds >= 2**64 are not supported on device")
    return s


def spawn_streams(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Host SeedSequence(seed).spawn(...)[offset:offset+n] PCG64 states ([n, 6] uint64)."""
    out = np.zeros((n, 6), dtype=np.uint64)
    _lib.check(_lib.load().lg_seed_streams(check_seed(seed), int(offset), int(n),
                                           out.ctypes.data_as(ctypes.c_void_p)))
    return out


class _Lease:
    """Exposes one pooled block as a new ndarray (``np.asarray(lease)``): the
    array's base is the lease, so the block goes back to its pool when the
    caller has dropped the array and every view of it."""
    __slots__ = ("__array_interface__", "block", "__weakref__")

    def __init__(self, block):
        self.block = block
        self.__array_interface__ = block.__array_interface__


class _HostPool:
    """Fresh output arrays without fresh pages. The reference returns new
    arrays every step (env.py:233); allocating them new makes every step
    page-fault and zero its whole output (16 GB for c5) before the copy.
    Here each step still returns arrays no earlier step returned and that the
    caller alone owns, but their memory is recycled from arrays the caller
    has released (at most ``keep`` idle blocks per key are retained)."""

    def __init__(self, keep: int = 2):
        self.keep = keep
        self.free: dict[Any, list] = {}

    def _release(self, key, block):
        lst = self.free.setdefault(key, [])
        if len(lst) < self.keep:
            lst.append(block)

    SMALL = 1 << 18  # below this, np.empty is cheaper than a lease (no page faults to save)

    def take(self, shape, dtype) -> np.ndarray:
        import weakref
        if int(np.prod(shape)) * np.dtype(dtype).itemsize < self.SMALL:
            return np.empty(shape, dtype)
        key = (tuple(shape), np.dtype(dtype).str)
        lst = self.free.get(key)
        block = lst.pop() if lst else np.empty(shape, dtype)
        lease = _Lease(block)
        weakref.finalize(lease, self._release, key, block)
        return np.asarray(lease)


class NumpyBatchEnv:
    """Reference-shaped facade: numpy in, numpy out (env.py:486-588).

    Every ``step`` goes through ``lg_step_host``: the host->device copy of the
    actions and the device->host copies of obs/reward/done/info happen inside
    the library call. With ``copy=True`` (the default) each step returns new
    arrays, as the reference does; their memory comes from arrays the caller
    has released (``_HostPool``), so a step does not fault in fresh pages.
    Pass ``pinned=True`` to stage through page-locked buffers (reused across
    steps; the arrays returned by ``step`` are then overwritten by the next
    step unless ``copy=True``).
    """

    def __init__(self, config: EnvConfig, n_envs: int, seed: int = 0, *, device: Any = None,
                 global_offset: int = 0, pinned: bool = False, copy: bool = True,
                 obs_dtype: str = "float32"):
        self.env = BatchEnv(config, n_envs, seed, device=device, global_offset=global_offset,
                            obs_dtype=obs_dtype)
        self.pinned = pinned
        self.copy = copy
        self._bufs = None
        self._args = None
        self._obs_seen = None
        self._pool = _HostPool()

    config = property(lambda self: self.env.config)
    n_envs = property(lambda self: self.env.n_envs)
    n_actions = property(lambda self: self.env.n_actions)
    observation_shape = property(lambda self: self.env.observation_shape)

    def _host(self):
        t = self.env._torch
        B = self.env.n_envs
        def mk(shape, dt):
            if self.pinned:
                return t.empty(shape, dtype=dt, pin_memory=True).numpy()
            return self._pool.take(shape, t.empty(0, dtype=dt).numpy().dtype)
        if self.env.obs_dtype == "bits":
            obs = mk(((B * int(np.prod(self.env.observation_shape)) + 31) // 32,), t.int32)
        else:
            obs = mk((B,) + self.env.observation_shape, t.uint8 if self.env.obs_dtype == "uint8" else t.float32)
        return {"obs": obs,
                "actions": mk((B,), t.int64), "reward": mk((B,), t.float64),
                "done": mk((B,), t.bool), "terminal": mk((B,), t.bool),
                "episode_reward": mk((B,), t.float64), "episode_length": mk((B,), t.int64),
                "episode_start_loss": mk((B,), t.float64), "final_loss": mk((B,), t.float64)}

    def reset(self) -> np.ndarray:
        return self.env.reset().cpu().numpy()

    def observe(self) -> np.ndarray:
        return self.env.observe().cpu().numpy()

    def step(self, actions):
        if not self.env._started:
            raise RuntimeError("reset() the batch before stepping")
        a = np.asarray(actions, dtype=np.int64)
        if a.shape != (self.n_envs,):
            raise ValueError(f"expected {self.n_envs} actions, got shape {a.shape}")
        if a.size and (a.min() < 0 or a.max() >= self.n_actions):
            raise ValueError("action id out of range")
        if self._bufs is None or (self.copy and not self.pinned):
            self._bufs = self._host()
            p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
            b = self._bufs
            # argument pointers built once per buffer set (small batches are latency-bound)
            self._args = (p(b["actions"]), p(b["obs"]), p(b["reward"]), p(b["done"]),
                          ctypes.byref(_lib.LgInfo(*[p(b[k]) for k in INFO_KEYS])))
        b = self._bufs
        if b["obs"] is not self._obs_seen:  # a caller may swap in its own obs array
            self._obs_seen = b["obs"]
            self._args = self._args[:1] + (b["obs"].ctypes.data_as(ctypes.c_void_p),) + self._args[2:]
        np.copyto(b["actions"], a)
        t = self.env._torch
        dev = self.env.device
        if t.cuda.current_device() == dev.index:
            _lib.check(_lib.load().lg_step_host(self.env.handle, *self._args, _stream(t, dev)))
        else:
            with t.cuda.device(dev):
                _lib.check(_lib.load().lg_step_host(self.env.handle, *self._args, _stream(t, dev)))
        info = {k: b[k] for k in INFO_KEYS}
        out = (b["obs"], b["reward"], b["done"], info)
        if self.copy and self.pinned:
            out = (b["obs"].copy(), b["reward"].copy(), b["done"].copy(),
                   {k: v.copy() for k, v in info.items()})
        return out

    def state_dict(self):
        return self.env.state_dict()

    def load_state_dict(self, state):
        self.env.load_state_dict(state)


def unpack_obs(bits, n_envs: int, shape, dtype=None):
    """Packed observation stream (obs_dtype="bits") -> [n_envs, C, OH, OW] 0/1 tensor."""
    import torch
    n = n_envs * int(np.prod(shape))
    b = bits.view(torch.uint8)[: (n + 7) // 8]
    sh = torch.arange(8, device=bits.device, dtype=torch.uint8)
    x = ((b[:, None] >> sh) & 1).reshape(-1)[:n]
    return x.reshape((n_envs,) + tuple(shape)).to(dtype or torch.float32)


__all__ = ["BatchEnv", "NumpyBatchEnv", "EnvConfig", "get_domain", "spawn_streams", "make_lg_config",
           "unpack_obs"]
