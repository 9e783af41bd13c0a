mkdir -p gpurun_out/r2s
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C3 > gpurun_out/r2s/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:map_assign -c 1 -o gpurun_out/r2s/map_c3 $C3 > gpurun_out/r2s/ncu.log 2>&1
ls -la gpurun_out/r2s
