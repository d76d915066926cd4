"""The binding a levelgen maintainer would add as ``levelgen/b200.py``.

Test infrastructure for INTEGRATION.md section 2: this file IS that stub,
verbatim, so tests/test_integration_stub.py can import it under a
``levelgen`` package (the reference's own, or the field-compatible mirror
``paper_2408_12525_b200.config.EnvConfig`` where the reference is absent, as
on the GPU box) and run it against the CPU oracle. It binds only the C ABI
(include/pcgrl_b200.h) with ctypes; nothing else of this repo.
"""
# levelgen/b200.py -- BatchEnv on a B200 through libpcgrl_b200.so
import ctypes
import os

import numpy as np
from .env import EnvConfig
from .grid import normalize_weights

_lib = ctypes.CDLL(os.environ.get("LEVELGEN_B200_LIB", "libpcgrl_b200.so"))
_P, _I64 = ctypes.c_void_p, ctypes.c_int64

class _Cfg(ctypes.Structure):                 # lg_config, include/pcgrl_b200.h
    _fields_ = [("domain", ctypes.c_int32), ("representation", ctypes.c_int32),
                ("max_h", ctypes.c_int32), ("max_w", ctypes.c_int32),
                ("obs_size", ctypes.c_int32), ("randomize_shape", ctypes.c_int32),
                ("init_weighted", ctypes.c_int32), ("n_pins", ctypes.c_int32),
                ("pins", ctypes.c_int32 * 16), ("n_ctrl", ctypes.c_int32),
                ("ctrl", ctypes.c_int32 * 8), ("max_steps", ctypes.c_int64),
                ("change_budget", ctypes.c_int64), ("det_metrics", ctypes.c_int32),
                ("obs_format", ctypes.c_int32), ("init_cdf", ctypes.c_double * 8),
                ("weights", ctypes.c_double * 8)]

class _Info(ctypes.Structure):                # lg_info
    _fields_ = [(k, _P) for k in ("terminal", "episode_reward", "episode_length",
                                  "episode_start_loss", "final_loss")]

_lib.lg_create.argtypes = [ctypes.POINTER(_Cfg), _I64, _I64, ctypes.c_uint64, ctypes.c_int,
                           ctypes.POINTER(_P)]
_lib.lg_reset.argtypes = [_P, _P, _P]
_lib.lg_step_host.argtypes = [_P, _P, _P, _P, _P, ctypes.POINTER(_Info), _P]
_lib.lg_destroy.argtypes = [_P]
_lib.lg_last_error.restype = ctypes.c_char_p

def _check(rc):
    if rc == 1: raise ValueError(_lib.lg_last_error().decode())
    if rc != 0: raise RuntimeError(_lib.lg_last_error().decode())

def _cfg(c: EnvConfig) -> _Cfg:
    d, x = c.domain_obj, _Cfg()
    x.domain = ("binary", "maze", "dungeon").index(d.name)
    x.max_h, x.max_w, x.obs_size = c.max_height, c.max_width, c.obs_size
    x.randomize_shape = c.randomize_shape
    x.init_weighted = (c.init_mode or d.default_init_mode) == "weighted"
    p = normalize_weights(d, c.init_weights or d.default_init_weights)   # grid.py:153-166
    cdf = p.cumsum(); cdf /= cdf[-1]                                      # Generator.choice
    for i, v in enumerate(cdf): x.init_cdf[i] = v
    x.n_pins = len(c.pinpoints)
    for i, t in enumerate(c.pinpoints): x.pins[i] = d.tile_id(t)
    ctrl = [i for i, m in enumerate(d.metric_names) if m in c.controllable]
    x.n_ctrl = len(ctrl)
    for i, m in enumerate(ctrl): x.ctrl[i] = m
    x.max_steps, x.change_budget = c.max_steps or 0, c.change_budget or 0
    x.det_metrics = c.deterministic_metrics
    x.obs_format = 0                          # LG_OBS_F32: the reference's float32 planes
    w = c.weights()
    for i, m in enumerate(d.metric_names): x.weights[i] = w[m]
    return x

class B200BatchEnv:
    """Drop-in for levelgen.env.BatchEnv (env.py:486-588), numpy in/out."""
    def __init__(self, config: EnvConfig, n_envs: int, seed: int = 0, device: int = 0):
        self.config, self.n_envs = config, n_envs
        self._h = _P()
        _check(_lib.lg_create(ctypes.byref(_cfg(config)), n_envs, 0, seed, device,
                              ctypes.byref(self._h)))
        c = config.observation_channels()
        self.observation_shape = (c, config.obs_size, config.obs_size)
        self._started = False

    n_actions = property(lambda self: self.config.n_actions)

    def reset(self):
        import torch                                   # device buffer for the reset obs
        obs = torch.empty((self.n_envs,) + self.observation_shape, device="cuda")
        _check(_lib.lg_reset(self._h, obs.data_ptr(), None))
        self._started = True
        return obs.cpu().numpy()

    def step(self, actions):
        if not self._started:
            raise RuntimeError("reset() the batch before stepping")
        a = np.ascontiguousarray(actions, dtype=np.int64)
        if a.shape != (self.n_envs,):
            raise ValueError(f"expected {self.n_envs} actions, got shape {a.shape}")
        if a.size and (a.min() < 0 or a.max() >= self.n_actions):
            raise ValueError("action id out of range")           # env.py:358-361
        B = self.n_envs
        obs = np.empty((B,) + self.observation_shape, np.float32)
        reward, done = np.empty(B, np.float64), np.empty(B, np.bool_)
        info = {"terminal": np.empty(B, np.bool_), "episode_reward": np.empty(B),
                "episode_length": np.empty(B, np.int64), "episode_start_loss": np.empty(B),
                "final_loss": np.empty(B)}
        p = lambda x: x.ctypes.data_as(_P)
        ci = _Info(*(p(info[k]) for k in ("terminal", "episode_reward", "episode_length",
                                          "episode_start_loss", "final_loss")))
        _check(_lib.lg_step_host(self._h, p(a), p(obs), p(reward), p(done), ctypes.byref(ci), None))
        return obs, reward, done, info

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lg_destroy(self._h)
