"""bench.py keeps the driver's JSON contract (one line; metric/value/unit, timing, roofline,
e2e, clocks, launches).  GPU: runs the real benchmark on the small config 1 workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line_contract():
    out = subprocess.run([sys.executable, "bench.py", "--config", "1", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline", "--spmv-nel", "0"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["1", "5"])
def test_bench_sharded_path_runs(config):
    """The --gpus N code path (NCCL process group, ShardedHomogenizer, packed all-gather, max-over-ranks
    timing) on one GPU via --sharded: linear (config 1) and finite strain (config 5)."""
    out = subprocess.run([sys.executable, "bench.py", "--config", config, "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline", "--spmv-nel", "0", "--no-companions", "--sharded"], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["config"]["parallelism"].startswith("rve-sharded")
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_reference_arm_json_line_runs_the_oracle():
    """--impl reference (the CPU oracle on the same workload) prints its own contract line."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tangents/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["value"] == d["value"]
