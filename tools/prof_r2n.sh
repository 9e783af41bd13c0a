# round 2: small-support Sinkhorn path -- tests, smoke, timing
mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q -p no:cacheprovider > gpurun_out/r2n/t_sparse.log 2>&1; tail -3 gpurun_out/r2n/t_sparse.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n/smoke.log 2>&1; tail -2 gpurun_out/r2n/smoke.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/b_c3.log 2>&1; tail -1 gpurun_out/r2n/b_c3.log | cut -c1-1500
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/b_c1.log 2>&1; tail -1 gpurun_out/r2n/b_c1.log | cut -c1-600
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pairs-api > gpurun_out/r2n/b_c3p.log 2>&1; tail -1 gpurun_out/r2n/b_c3p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pairs_api', d.get('pairs_api'))"
