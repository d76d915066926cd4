"""Host side of the packed observation transfer (lg_unpack_host = the
expansion lg_step_host runs after the copy), on CPU against numpy: sizes
around the byte/word/chunk edges, both output formats, the multi-threaded
path (>= 4 MB of output) and unaligned destinations."""
import ctypes

import numpy as np
import pytest

from paper_2408_12525_b200 import _lib


def unpack_ref(words, n, dtype):
    b = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
    return b.astype(dtype)


@pytest.mark.parametrize("fmt,dtype", [(0, np.float32), (1, np.uint8)])
@pytest.mark.parametrize("n", [0, 1, 7, 8, 31, 33, 1000, 3844 * 37, 5_000_003])
@pytest.mark.parametrize("misalign", [0, 4, 8, 20])
def test_unpack_matches_numpy(fmt, dtype, n, misalign):
    lib = _lib.load()
    rng = np.random.default_rng(n + misalign)
    words = rng.integers(0, 2 ** 32, size=(n + 31) // 32 + 1, dtype=np.uint64).astype(np.uint32)
    item = np.dtype(dtype).itemsize
    raw = np.full(n * item + 64, 0xAB, dtype=np.uint8)
    off = (misalign - raw.ctypes.data) % 64
    out = raw[off:off + n * item].view(dtype)
    assert n == 0 or out.ctypes.data % 64 == misalign % 64
    _lib.check(lib.lg_unpack_host(words.ctypes.data_as(ctypes.c_void_p), n,
                                  out.ctypes.data_as(ctypes.c_void_p), fmt))
    assert np.array_equal(out, unpack_ref(words, n, dtype))
    assert (raw[:off] == 0xAB).all() and (raw[off + n * item:] == 0xAB).all()  # nothing outside


def test_unpack_rejects_bad_arguments():
    lib = _lib.load()
    w = np.zeros(4, np.uint32)
    o = np.zeros(8, np.float32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    with pytest.raises(ValueError):
        _lib.check(lib.lg_unpack_host(p(w), 8, p(o), 2))
    with pytest.raises(ValueError):
        _lib.check(lib.lg_unpack_host(p(w), -1, p(o), 0))
