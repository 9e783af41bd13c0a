"""bench.py's JSON-line contract (the driver parses it): one line with the required keys, on a
small workload, for our arm and the reference arm (the oracle)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.sparse_path,   # bench.py refuses ASOT_SPARSE
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
            "gpu_launches", "clocks")


def run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_ours():
    d = run("--config", "c2", "--n-dist", "200", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
            "--cpu-budget", "1")
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    rf = d["roofline"]
    assert rf["bound"] in ("tensor", "alu", "hbm") and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "workload" in d["config"]
    # tensor-core kernels: the in-kernel clock probe gives the clock the timed launches ran at
    assert rf["bound"] == "tensor"
    assert 300.0 < rf["effective_sm_mhz"] < 2500.0
    assert abs(rf["frac_of_nominal_effective"] * rf["nominal_peak_at_effective_clock"] - rf["achieved"]) < 1e-6 * rf["achieved"]

