"""B200-native batched PCGRL env step (arXiv 2408.12525), drop-in for levelgen's BatchEnv.

Host code is Python; the step itself is hand-written sm_100a CUDA behind the
C ABI in include/pcgrl_b200.h (libpcgrl_b200.so, built in-tree by
``python -m paper_2408_12525_b200.build``).
"""
from .config import EnvConfig
from .tiles import BINARY, DOMAINS, DUNGEON, MAZE, Domain, get_domain

__all__ = ["EnvConfig", "Domain", "BINARY", "MAZE", "DUNGEON", "DOMAINS", "get_domain",
           "BatchEnv", "NumpyBatchEnv"]


def __getattr__(name):
    if name in ("BatchEnv", "NumpyBatchEnv", "spawn_streams"):
        from . import env
        return getattr(env, name)
    raise AttributeError(name)
