# round 2: small-support Sinkhorn path -- tests, timing, ncu of the sparse kernel at c3
mkdir -p gpurun_out/r2o
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -p no:cacheprovider > gpurun_out/r2o/t_sparse.log 2>&1; tail -3 gpurun_out/r2o/t_sparse.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2o/b_c3.log 2>&1; tail -1 gpurun_out/r2o/b_c3.log | cut -c1-400
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_sparse" -c 1 -o gpurun_out/r2o/sparse_c3 $C3 > gpurun_out/r2o/ncu.log 2>&1; tail -1 gpurun_out/r2o/ncu.log
