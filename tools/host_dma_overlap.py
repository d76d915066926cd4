"""Can host memory absorb the packed-bit expansion (CPU threads, NT stores) and
a PCIe D2H DMA at the same time? Times each alone and both together.
    python tools/host_dma_overlap.py"""
import ctypes
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_12525_b200 import _lib  # noqa: E402

lib = _lib.load()
n_el = 3 * 1024 ** 3 // 4          # 3 GB of float32 output from the expansion
bits = np.random.default_rng(0).integers(0, 2**32, size=(n_el + 31) // 32, dtype=np.uint32)
dst = torch.empty(n_el, dtype=torch.float32).pin_memory().numpy()
dma_bytes = 1024 ** 3
src = torch.empty(dma_bytes // 4, dtype=torch.float32, device="cuda")
hdst = torch.empty(dma_bytes // 4, dtype=torch.float32).pin_memory()


def expand():
    _lib.check(lib.lg_unpack_host(bits.ctypes.data_as(ctypes.c_void_p), n_el, dst.ctypes.data_as(ctypes.c_void_p), 0))


def dma():
    hdst.copy_(src, non_blocking=False)


for f in (expand, dma):
    f()
t0 = time.perf_counter(); expand(); t_e = time.perf_counter() - t0
t0 = time.perf_counter(); dma(); t_d = time.perf_counter() - t0
th = threading.Thread(target=dma)
t0 = time.perf_counter(); th.start(); expand(); th.join(); t_b = time.perf_counter() - t0
print(f"expand alone {n_el * 4 / t_e / 1e9:.1f} GB/s ({t_e*1e3:.0f} ms); dma alone {dma_bytes / t_d / 1e9:.1f} GB/s "
      f"({t_d*1e3:.0f} ms); both {t_b*1e3:.0f} ms -> {(n_el * 4 + dma_bytes) / t_b / 1e9:.1f} GB/s combined")
