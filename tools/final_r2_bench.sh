# round-2 final: bench lines (one JSON line each) + ncu evidence (outputs under gpurun_out/final/)
mkdir -p gpurun_out/final/bench
B="python bench.py"
run() { name=$1; shift; $B "$@" > gpurun_out/final/bench/$name.log 2>&1; tail -1 gpurun_out/final/bench/$name.log > gpurun_out/final/bench/$name.json; python -c "import json; d=json.load(open('gpurun_out/final/bench/$name.json')); print('$name', d.get('value'), d.get('ms_per_step'), d.get('roofline',{}).get('kernel','')[:40], d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null || echo "$name FAILED"; }
run default
run reference --impl reference --steps 3 --warmup 3
run c1_tf32 --config c1 --steps 20 --warmup 5 --no-cpu-baseline
run c2_tf32 --config c2 --steps 20 --warmup 5 --no-cpu-baseline --pairs-api
run c3_tf32_pairs --steps 10 --warmup 3 --no-cpu-baseline --pairs-api
run c4_tf32 --config c4 --steps 3 --warmup 3 --no-cpu-baseline
run c5_tf32 --config c5 --steps 3 --warmup 3 --no-cpu-baseline
run c2_fp32 --config c2 --precision fp32 --steps 10 --warmup 3 --no-cpu-baseline --pairs-api
run c3_fp32 --precision fp32 --steps 10 --warmup 3 --no-cpu-baseline --pairs-api
run c4_fp32 --config c4 --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline
run c5_fp32 --config c5 --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1
run c3_ml --mapping ml --steps 5 --warmup 3 --no-cpu-baseline
run c3_dl --mapping dl --steps 5 --warmup 3 --no-cpu-baseline
run c5_ml --config c5 --mapping ml --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1
run c5_dl --config c5 --mapping dl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1
run c3_kmeans --anchors kmeans --steps 5 --warmup 3 --no-cpu-baseline
run c3_eot --baseline eot --steps 5 --warmup 3
run c2_exact --config c2 --exact --steps 5 --warmup 3 --no-cpu-baseline
run c2_bounds --config c2 --bounds --steps 5 --warmup 3 --no-cpu-baseline
# ncu: the launch list of the default command, then full captures of the top kernels
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/c3_launches.csv $C3 > gpurun_out/final/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_sparse|map_assign" -c 2 -o gpurun_out/final/sparse_c3 $C3 > gpurun_out/final/ncu_c3.log 2>&1
C2="python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_tc_kernel" -c 1 -o gpurun_out/final/tc_c2 $C2 > gpurun_out/final/ncu_c2.log 2>&1
ls -la gpurun_out/final
