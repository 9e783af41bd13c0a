# small-support kernels with paired reciprocals (one MUFU per two divides, per-pair rerun test):
# sparse tests + c3 bench + launch list + full ncu captures of the rect class kernels
mkdir -p gpurun_out/r2pair
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_pair_bucket.py -q -p no:cacheprovider > gpurun_out/r2pair/t_sparse.log 2>&1; tail -1 gpurun_out/r2pair/t_sparse.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2pair/b_c3.log 2>&1; tail -1 gpurun_out/r2pair/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'])"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2pair/c3_launches.csv $C3 > gpurun_out/r2pair/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_sparse_rect" -c 6 -o gpurun_out/r2pair/rect_c3 $C3 > gpurun_out/r2pair/ncu_full.log 2>&1
ls gpurun_out/r2pair
