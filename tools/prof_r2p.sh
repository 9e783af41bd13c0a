# round 2: small-support path -- the whole GPU suite, smoke, default bench line, ncu evidence
mkdir -p gpurun_out/r2p
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2p/gputest.log 2>&1; tail -3 gpurun_out/r2p/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p/smoke.log 2>&1; tail -2 gpurun_out/r2p/smoke.log
python bench.py > gpurun_out/r2p/bench_default.log 2>&1; tail -1 gpurun_out/r2p/bench_default.log > gpurun_out/r2p/bench_default.json; cut -c1-300 gpurun_out/r2p/bench_default.json
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p/c3_launches.csv $C3 > gpurun_out/r2p/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sinkhorn_sparse|support_kernel|gibbs_rows" -c 3 -o gpurun_out/r2p/sparse_c3 $C3 > gpurun_out/r2p/ncu_full.log 2>&1; tail -1 gpurun_out/r2p/ncu_full.log
