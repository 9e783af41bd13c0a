# ncu evidence for profiles/ (run under gpurun; each capture only after its command ran clean)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/pre.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_tc2 -c 1 -o gpurun_out/tc2_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --n-dist 600 > gpurun_out/ncu_tc2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_tc3 -c 1 -o gpurun_out/tc3_c2 python bench.py --config c2 --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --n-dist 600 > gpurun_out/ncu_tc3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_simt -c 1 -o gpurun_out/simt_c3 python bench.py --config c3 --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --n-dist 300 > gpurun_out/ncu_simt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:exact_pairs -c 1 -o gpurun_out/exact_c4 python bench.py --config c4 --exact --exact-pairs 4000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --n-dist 600 > gpurun_out/ncu_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_tc_kernel -c 1 -o gpurun_out/tc_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_tc.log 2>&1
ls -la gpurun_out
