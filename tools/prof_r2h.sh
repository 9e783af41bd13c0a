mkdir -p gpurun_out/r2c1
for i in 1 2; do python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c1/c1_$i.log 2>&1; tail -1 gpurun_out/r2c1/c1_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value']/1e6, d['ms_per_step'], d['roofline'].get('kernel_ms_per_launch'))"; done
python -m pytest tests/test_gpu_ratio.py tests/test_gpu_edge.py -x -q 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or warp or simt" 2>&1 | tail -2
C="python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:sinkhorn_warp -c 1 -o gpurun_out/r2c1/warp_c1b $C > gpurun_out/r2c1/ncu.log 2>&1
