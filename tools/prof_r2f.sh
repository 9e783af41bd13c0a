mkdir -p gpurun_out/r2pb2
python -m pytest tests/test_gpu_pair_bucket.py -x -q > gpurun_out/r2pb2/tests_new.log 2>&1; tail -3 gpurun_out/r2pb2/tests_new.log
python -m pytest tests/test_gpu_parity.py -x -q -k "pair" > gpurun_out/r2pb2/tests_old.log 2>&1; tail -3 gpurun_out/r2pb2/tests_old.log
for c in c2 c3; do for p in fp32; do python bench.py --config $c --precision $p --steps 5 --warmup 3 --no-cpu-baseline --pairs-api > gpurun_out/r2pb2/bench_${c}_$p.log 2>&1; tail -1 gpurun_out/r2pb2/bench_${c}_$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $p', d['value']/1e6, d['pairs_api'])"; done; done
