"""bench.py keeps the driver's JSON-line contract: the reference arm on the
host cores (CPU tier) and the B200 arm, single-rank and two ranks folded onto
one GPU (the multi-rank timing path: barrier, max over ranks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl"}


def _json_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1",
                        "--steps", "1", "--warmup", "3", "--cpu-seconds", "0.3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _json_line(r.stdout)
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference" and line["value"] > 0 and line["warmup"] >= 3
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference")
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["value"] == line["value"]


@pytest.mark.gpu
def test_b200_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--secondary", "c1m",
                        "--steps", "3", "--warmup", "3", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _json_line(r.stdout)
    assert BASE_KEYS <= set(line) and line["impl"] == "b200" and line["n_gpus"] == 1
    assert line["value"] > 0 and line["gpu_launches"] >= 3
    roof = line["roofline"]
    assert roof["bound"] in ("tensor", "hbm") and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
    assert "c1m" in line["per_dim"] and line["per_dim"]["c1m"]["value"] > 0


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_time_sharded():
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", "bench.py", "--gpus", "2", "--workload", "c1",
                        "--secondary", "", "--steps", "3", "--warmup", "3", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0
