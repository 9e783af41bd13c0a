python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --config c2 --precision fp32 --steps 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_fp32.log 2>&1
python bench.py --config c3 --precision fp32 --steps 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_fp32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:soft_map -c 1 -o gpurun_out/soft_dl_c3 python bench.py --config c3 --mapping dl --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_dl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_simt -c 1 -o gpurun_out/simt_c2 python bench.py --config c2 --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_simt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:eot_pairs -c 1 -o gpurun_out/eot_c3 python bench.py --config c3 --baseline eot --eot-pairs 4000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_eot.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c3_dl_launches.csv python bench.py --config c3 --mapping dl --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_dl_launch.log 2>&1
for f in gpurun_out/bench_c*_fp32.log; do tail -n 1 $f | cut -c 1-900; done
