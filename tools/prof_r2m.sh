# round 2: ML on tcgen05, two-pass GEMM 2 with the butterfly histogram
mkdir -p gpurun_out/r2m
timeout 600 python -m pytest tests/test_gpu_soft.py -x -q -p no:cacheprovider > gpurun_out/r2m/t_soft.log 2>&1; tail -2 gpurun_out/r2m/t_soft.log
P='import json,sys; d=json.loads(sys.stdin.read()); m=d["mapping"]; print(sys.argv[1], d["value"], m["ms_per_launch"], m.get("fp32_pipe_frac", m.get("bf16_frac")))'
python bench.py --mapping ml --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_ml.log 2>&1; tail -1 gpurun_out/r2m/b_ml.log | python -c "$P" ml
python bench.py --config c5 --mapping ml --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2m/b_c5ml.log 2>&1; tail -1 gpurun_out/r2m/b_c5ml.log | python -c "$P" c5ml
python bench.py --config c2 --mapping ml --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_c2ml.log 2>&1; tail -1 gpurun_out/r2m/b_c2ml.log | python -c "$P" c2ml
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --mapping ml"
ncu --set full --clock-control none --import-source on -k regex:"soft_ml_tc" -c 1 -o gpurun_out/r2m/ml_c3 $C3 > gpurun_out/r2m/ncu_ml.log 2>&1; tail -1 gpurun_out/r2m/ncu_ml.log
