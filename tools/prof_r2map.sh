# exact mapping kernel: refine reads the anchors from the CTA's shared copy -- mapping tests
# (bit-exact incl. c3 all points, c5 10%), c3 bench, ncu of the list-mode exact pass
mkdir -p gpurun_out/r2map
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -k mapping -q -p no:cacheprovider > gpurun_out/r2map/t_map.log 2>&1; tail -1 gpurun_out/r2map/t_map.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2map/b_c3.log 2>&1; tail -1 gpurun_out/r2map/b_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['mapping']['ms_per_launch'])"
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2map/b_c5.log 2>&1; tail -1 gpurun_out/r2map/b_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['mapping']['ms_per_launch'])"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2map/c3_launches.csv $C3 > gpurun_out/r2map/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"map_assign|map_tc_kernel" -c 4 -o gpurun_out/r2map/map_c3 $C3 > gpurun_out/r2map/ncu_full.log 2>&1
ls gpurun_out/r2map
