# round 2: map_assign 32-lane layout (K >= 128) + ML on tcgen05 (column pass batched)
mkdir -p gpurun_out/r2l
python -m pytest tests/test_gpu_parity.py -k "mapping" -x -q -p no:cacheprovider > gpurun_out/r2l/t_map.log 2>&1; tail -2 gpurun_out/r2l/t_map.log
timeout 600 python -m pytest tests/test_gpu_soft.py tests/test_gpu_kmeans.py -x -q -p no:cacheprovider > gpurun_out/r2l/t_soft.log 2>&1; tail -2 gpurun_out/r2l/t_soft.log
P='import json,sys; d=json.loads(sys.stdin.read()); m=d["mapping"]; print(sys.argv[1], d["value"], m["ms_per_launch"], m.get("fp32_pipe_frac", m.get("bf16_frac")))'
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l/b_c3.log 2>&1; tail -1 gpurun_out/r2l/b_c3.log | python -c "$P" c3
python bench.py --mapping ml --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l/b_ml.log 2>&1; tail -1 gpurun_out/r2l/b_ml.log | python -c "$P" ml
python bench.py --config c5 --mapping ml --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2l/b_c5ml.log 2>&1; tail -1 gpurun_out/r2l/b_c5ml.log | python -c "$P" c5ml
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2l/b_c5.log 2>&1; tail -1 gpurun_out/r2l/b_c5.log | python -c "$P" c5
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l/b_c2.log 2>&1; tail -1 gpurun_out/r2l/b_c2.log | python -c "$P" c2
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"map_assign" -c 1 -o gpurun_out/r2l/map_c3 $C3 > gpurun_out/r2l/ncu_map.log 2>&1; tail -1 gpurun_out/r2l/ncu_map.log
ncu --set full --clock-control none --import-source on -k regex:"soft_ml_tc" -c 1 -o gpurun_out/r2l/ml_c3 $C3 --mapping ml > gpurun_out/r2l/ncu_ml.log 2>&1; tail -1 gpurun_out/r2l/ncu_ml.log
