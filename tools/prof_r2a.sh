set -x
mkdir -p gpurun_out/r2p
C5="python bench.py --config c5 --n-dist 300 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
C3F="python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C5 > gpurun_out/r2p/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn_tc4 -c 1 -o gpurun_out/r2p/tc4_c5 $C5 > gpurun_out/r2p/ncu_c5.log 2>&1
$C3F > gpurun_out/r2p/plain_c3f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn_tc6 -c 1 -o gpurun_out/r2p/tc6_c3 $C3F > gpurun_out/r2p/ncu_c3f.log 2>&1
$C3 > gpurun_out/r2p/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_tc2|map_assign" -c 2 -o gpurun_out/r2p/tc2_c3 $C3 > gpurun_out/r2p/ncu_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p/c3_launches.csv $C3 > gpurun_out/r2p/ncu_c3_launch.log 2>&1
ls -la gpurun_out/r2p
