# ncu: the tensor-core mapping kernel and the list refine at c3
mkdir -p gpurun_out/r2u
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"map_tc_kernel|map_assign" -c 2 -o gpurun_out/r2u/maptc_c3 $C3 > gpurun_out/r2u/ncu.log 2>&1; tail -1 gpurun_out/r2u/ncu.log
