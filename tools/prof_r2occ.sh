# small-support kernels at more CTAs per SM (8 / 8 / 6 / 6 / 5 / 4 for 4x4 .. 8x8; the hot loops
# stay spill-free): sparse tests + c3 bench + launch list + ncu of the rect kernels
mkdir -p gpurun_out/r2o
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_pair_bucket.py -q -p no:cacheprovider > gpurun_out/r2o/t_sparse.log 2>&1; tail -1 gpurun_out/r2o/t_sparse.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2o/b_c3.log 2>&1; tail -1 gpurun_out/r2o/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'])"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o/c3_launches.csv $C3 > gpurun_out/r2o/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_sparse_rect" -c 6 -o gpurun_out/r2o/rect_c3 $C3 > gpurun_out/r2o/ncu_full.log 2>&1
ls gpurun_out/r2o
