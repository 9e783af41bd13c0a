# small-support kernels A/B: sparse tests + c3 bench + launch list
mkdir -p gpurun_out/r2w
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -p no:cacheprovider > gpurun_out/r2w/t_sparse.log 2>&1; tail -1 gpurun_out/r2w/t_sparse.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2w/b_c3.log 2>&1; tail -1 gpurun_out/r2w/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'])"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2w/c3_launches.csv $C3 > gpurun_out/r2w/ncu_launch.log 2>&1
