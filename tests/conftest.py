import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    # the product library is built in-tree (nvcc cross-compiles without a GPU)
    from paper_2408_12525_b200 import build
    if build.stale():
        try:
            build.build()
        except Exception as exc:  # surfaced by the ABI tests
            sys.stderr.write(f"[conftest] CUDA build failed: {exc}\n")
    from oracle import oracle
    oracle.build()
