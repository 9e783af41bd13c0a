mkdir -p gpurun_out/r2q
C5="python bench.py --config c5 --n-dist 300 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C5 > gpurun_out/r2q/plain_c5.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:sinkhorn_tc4 -c 1 --csv --log-file gpurun_out/r2q/tc4_c5_metrics.csv $C5 > gpurun_out/r2q/ncu.log 2>&1
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q/bench_c5.log 2>&1
cat gpurun_out/r2q/tc4_c5_metrics.csv | tail -8
