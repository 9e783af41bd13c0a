# mapping: expanded form on the 32-lane layout -- parity + timing
mkdir -p gpurun_out/r2r
python -m pytest tests/test_gpu_parity.py -k "mapping" -x -q -p no:cacheprovider > gpurun_out/r2r/t_map.log 2>&1; tail -2 gpurun_out/r2r/t_map.log
timeout 900 python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "map or assign or kmeans" > gpurun_out/r2r/t_full.log 2>&1; tail -2 gpurun_out/r2r/t_full.log
P='import json,sys; d=json.loads(sys.stdin.read()); m=d["mapping"]; print(sys.argv[1], d["value"], m["ms_per_launch"], m.get("fp32_pipe_frac"))'
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2r/b_c3.log 2>&1; tail -1 gpurun_out/r2r/b_c3.log | python -c "$P" c3
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2r/b_c5.log 2>&1; tail -1 gpurun_out/r2r/b_c5.log | python -c "$P" c5
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2r/b_c4.log 2>&1; tail -1 gpurun_out/r2r/b_c4.log | python -c "$P" c4
