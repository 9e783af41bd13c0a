mkdir -p gpurun_out/r2dl3
C="python bench.py --config c3 --mapping dl --n-dist 300 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C > gpurun_out/r2dl3/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:soft_dl_tc -c 1 -o gpurun_out/r2dl3/dltc_c3 $C > gpurun_out/r2dl3/ncu.log 2>&1
ls gpurun_out/r2dl3
