mkdir -p gpurun_out/r2z5
python -m pytest tests/test_gpu_soft.py -x -q > gpurun_out/r2z5/tests.log 2>&1; tail -3 gpurun_out/r2z5/tests.log
for c in c3 c5; do python bench.py --config $c --mapping dl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2z5/bench_$c.log 2>&1; tail -1 gpurun_out/r2z5/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d.get('mapping',{}).get('ms_per_launch'))"; done
C="python bench.py --config c5 --mapping dl --n-dist 60 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$C > gpurun_out/r2z5/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:soft_dl_tc -c 1 -o gpurun_out/r2z5/dltc_c5 $C > gpurun_out/r2z5/ncu.log 2>&1
ls gpurun_out/r2z5
