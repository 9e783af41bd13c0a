# small-support kernel A/B: bench c3 only
mkdir -p gpurun_out/r2q
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2q/b_c3.log 2>&1; tail -1 gpurun_out/r2q/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'])"
