"""Diagnostic: kernel time in normal / MMA-only (no epilogue) / epilogue-only (no MMA) modes."""
import json, os, subprocess, sys
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
extra = sys.argv[2:]
for mode in ("0", "1", "2"):
    env = dict(os.environ, ASOT_TC_DEBUG_MODE=mode)
    out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "3", "--warmup", "3",
                          "--e2e-steps", "1", "--no-cpu-baseline", *extra], env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        print(cfg, "mode", mode, "kernel ms", round(d["roofline"]["kernel_ms_per_launch"], 3), flush=True)
    except Exception:
        print(mode, "failed", out.stderr[-400:], flush=True)
