"""bench.py --impl reference (this tier's reference arm = the fp64 oracle on the host cores): one
JSON line, the same metric / unit / config as our arm, whole-job pairs/s extrapolated from pooled
per-point mapping and per-pair Sinkhorn times.  Runs on CPU (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_reference_arm():
    d = run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1", "--ref-pairs", "16",
            "--ref-dists", "8")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "pairs/s"
    assert d["higher_is_better"] is True and d["n_gpus"] == 1 and d["steps"] == 2
    assert "workload" in d["config"] and d["config"]["pairs"] == 2016
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # whole-job throughput: the 2,016-pair c1 matrix in well under a minute of oracle time
    assert d["value"] * 60 > d["config"]["pairs"]
