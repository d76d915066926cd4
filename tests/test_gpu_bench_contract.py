"""bench.py keeps the driver's JSON contract (one line, required keys), on a
small c5-shaped run (needs a B200)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_ours_line():
    d = _run("--envs", "8192", "--steps", "3", "--warmup", "3", "--no-policy", "--cpu-envs", "256",
             "--cpu-seconds", "0.5")
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["gpu_launches"] == 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8192 * 8 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_line():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "3", "--cpu-envs", "256")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_two_rank_code_path_functional():
    """The N > 1 path of bench.py under torchrun (2 ranks): shards, barriers,
    the side-stream stats all-reduce every S steps, max-over-ranks timing and
    one JSON line from rank 0. A functional test on a one-GPU box: both ranks
    on cuda:0 with the gloo backend (LG_BENCH_SAME_DEVICE / LG_BENCH_BACKEND),
    never a measurement."""
    env = dict(os.environ, LG_BENCH_SAME_DEVICE="1", LG_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--envs", "16384", "--steps", "10", "--warmup", "3", "--stats-every", "5", "--no-policy", "--no-u8",
           "--cpu-envs", "256", "--cpu-seconds", "0.5"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_envs"] == 16384 and d["config"]["envs_per_gpu"] == 8192
    assert d["stats_all_reduce"]["count"] == 2 and d["host"]["comm"] == "gloo x2"
    assert d["cpu_baseline"]["value"] > 0 and d["e2e"]["value"] > 0
    assert "communicator of 2 ranks" in out.stderr
