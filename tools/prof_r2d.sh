mkdir -p gpurun_out/r2y
C="python bench.py --config c5 --mapping dl --n-dist 60 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C > gpurun_out/r2y/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:soft_dl_tc -c 1 -o gpurun_out/r2y/dltc_c5 $C > gpurun_out/r2y/ncu.log 2>&1
ls -la gpurun_out/r2y
