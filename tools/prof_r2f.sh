mkdir -p gpurun_out/r2pb
python -m pytest tests/test_gpu_pair_bucket.py -x -q > gpurun_out/r2pb/tests_new.log 2>&1; tail -3 gpurun_out/r2pb/tests_new.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_ratio.py tests/test_gpu_edge.py -x -q > gpurun_out/r2pb/tests_old.log 2>&1; tail -3 gpurun_out/r2pb/tests_old.log
for c in c2 c3; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --pairs-api > gpurun_out/r2pb/bench_$c.log 2>&1; tail -1 gpurun_out/r2pb/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value']/1e6, d['pairs_api'])"; done
