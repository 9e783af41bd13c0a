# ncu: the dominant small-support class kernel (6 x 6 form) at c3
mkdir -p gpurun_out/r2v
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k sinkhorn_sparse_class_kernel --launch-skip 1 -c 1 -o gpurun_out/r2v/cls6_c3 $C3 > gpurun_out/r2v/ncu.log 2>&1; tail -1 gpurun_out/r2v/ncu.log
