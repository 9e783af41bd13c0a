mkdir -p gpurun_out/r2pb3
python -m pytest tests/test_gpu_pair_bucket.py -x -q > gpurun_out/r2pb3/tests_new.log 2>&1; tail -3 gpurun_out/r2pb3/tests_new.log
for p in tf32 fp32; do python bench.py --config c5 --precision $p --n-dist 1000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --pairs-api > gpurun_out/r2pb3/bench_c5_$p.log 2>&1; tail -1 gpurun_out/r2pb3/bench_c5_$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $p', d['value']/1e6, d['pairs_api'])"; done
