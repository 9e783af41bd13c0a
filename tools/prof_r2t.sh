# tensor-core mapping (R#37): parity (both paths) + timing
mkdir -p gpurun_out/r2t
timeout 900 python -m pytest tests/test_gpu_parity.py -k "mapping" -x -q -p no:cacheprovider > gpurun_out/r2t/t_map.log 2>&1; tail -2 gpurun_out/r2t/t_map.log
timeout 1200 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "mapping" > gpurun_out/r2t/t_full.log 2>&1; tail -2 gpurun_out/r2t/t_full.log
P='import json,sys; d=json.loads(sys.stdin.read()); m=d["mapping"]; print(sys.argv[1], d["value"], d["ms_per_step"], m["ms_per_launch"])'
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2t/b_c3.log 2>&1; tail -1 gpurun_out/r2t/b_c3.log | python -c "$P" c3
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2t/b_c5.log 2>&1; tail -1 gpurun_out/r2t/b_c5.log | python -c "$P" c5
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2t/b_c2.log 2>&1; tail -1 gpurun_out/r2t/b_c2.log | python -c "$P" c2
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t/c3_launches.csv $C3 > gpurun_out/r2t/ncu_launch.log 2>&1; tail -1 gpurun_out/r2t/ncu_launch.log | cut -c1-100
