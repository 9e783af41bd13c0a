# round-2 late: histogram kernel with the running bin sum held in a register (plus the prefetched batches).
mkdir -p gpurun_out/r2h2
python -m pytest tests/test_gpu_sparse.py tests/test_gpu_edge.py tests/test_gpu_bench_contract.py -m gpu -q -p no:cacheprovider > gpurun_out/r2h2/gputest_a.log 2>&1; tail -3 gpurun_out/r2h2/gputest_a.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -q -p no:cacheprovider -k "mapping or map_ws or nccl or c3" > gpurun_out/r2h2/gputest_b.log 2>&1; tail -3 gpurun_out/r2h2/gputest_b.log
for i in 1 2 3; do
python bench.py --no-cpu-baseline > gpurun_out/r2h2/bench_default_$i.log 2>&1; tail -1 gpurun_out/r2h2/bench_default_$i.log > gpurun_out/r2h2/bench_default_$i.json
python -c "import json; d=json.load(open('gpurun_out/r2h2/bench_default_$i.json')); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['e2e']['value'], d['clocks'])"
done
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h2/c3_launches.csv $C3 > gpurun_out/r2h2/ncu_launch.log 2>&1
