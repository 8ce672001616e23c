"""bench.py's JSON line keeps the driver's contract (keys, types, the
roofline / cpu_baseline / e2e / clocks objects) on a short GPU run, and the
reference arm prints its own line."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run("--steps", "3", "--warmup", "3", "--no-frame", "--no-cpu-baseline",
             "--n", str(1 << 20))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 * max(1.0, r["frac"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] >= 3


def test_reference_arm_line():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--n", str(1 << 20))
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_two_ranks_line():
    """bench.py under torchrun with 2 ranks (gloo, both on this GPU): one
    JSON line from rank 0 with n_gpus = 2, the sharded frame's replicas
    identical; the reference arm prints once."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, NIRC_DIST_BACKEND="gloo")

    def run(port, *args):
        out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                              "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                              "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                              "--gpus", "2", *args],
                             capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, out.stdout[-2000:]
        return json.loads(lines[0])

    # (torchrun's own parser would take bench.py's --n for one of its options)
    d = run(29611, "--steps", "3", "--warmup", "3", "--frame-steps", "2", "--no-extra-frames",
            "--no-cpu-baseline")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["frame_1080p"]["replicas_identical"] is True
    r = run(29612, "--impl", "reference", "--steps", "1", "--warmup", "0")
    assert r["impl"] == "reference" and r["n_gpus"] == 2
