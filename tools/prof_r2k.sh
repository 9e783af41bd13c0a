# round 2: dot-form mapping kernel + ML on tcgen05 -- targeted GPU tests and bench lines
mkdir -p gpurun_out/r2k
python -m pytest tests/test_gpu_parity.py -k "mapping" -x -q -p no:cacheprovider > gpurun_out/r2k/t_map.log 2>&1; tail -2 gpurun_out/r2k/t_map.log
timeout 600 python -m pytest tests/test_gpu_soft.py tests/test_gpu_eot.py tests/test_gpu_kmeans.py -x -q -p no:cacheprovider > gpurun_out/r2k/t_soft.log 2>&1; tail -2 gpurun_out/r2k/t_soft.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k/b_c3.log 2>&1; tail -1 gpurun_out/r2k/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['mapping'])"
python bench.py --mapping ml --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2k/b_ml.log 2>&1; tail -1 gpurun_out/r2k/b_ml.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ml', d['value'], d['mapping'])"
python bench.py --config c5 --mapping ml --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2k/b_c5ml.log 2>&1; tail -1 gpurun_out/r2k/b_c5ml.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5ml', d['value'], d['mapping'])"
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2k/b_c5.log 2>&1; tail -1 gpurun_out/r2k/b_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['mapping'])"
