mkdir -p gpurun_out/r2c1
C="python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline"
$C > gpurun_out/r2c1/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn_warp -c 1 -o gpurun_out/r2c1/warp_c1 $C > gpurun_out/r2c1/ncu.log 2>&1
