"""Diagnostic: time the TC Sinkhorn kernel on c2 in normal / MMA-only / epilogue-only modes."""
import os, subprocess, sys, json
for mode in ("0", "1", "2"):
    env = dict(os.environ, ASOT_TC_DEBUG_MODE=mode)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--e2e-steps", "1",
                          "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(mode, "kernel ms", d["roofline"]["kernel_ms_per_launch"], flush=True)
    except Exception:
        print(mode, "failed", out.stderr[-500:], flush=True)
