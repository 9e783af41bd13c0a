# round-2 closing check: the GPU suite + smoke, then the default line, the reference arm and the
# launch list on the final library (outputs under gpurun_out/final_c/)
mkdir -p gpurun_out/final_c
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_c/gputest.log 2>&1; tail -3 gpurun_out/final_c/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_c/smoke.log 2>&1; tail -1 gpurun_out/final_c/smoke.log
python bench.py > gpurun_out/final_c/default.log 2>&1; tail -1 gpurun_out/final_c/default.log > gpurun_out/final_c/default.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_c/reference.log 2>&1; tail -1 gpurun_out/final_c/reference.log > gpurun_out/final_c/reference.json
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c/c5_tf32.log 2>&1; tail -1 gpurun_out/final_c/c5_tf32.log > gpurun_out/final_c/c5_tf32.json
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final_c/c2_tf32.log 2>&1; tail -1 gpurun_out/final_c/c2_tf32.log > gpurun_out/final_c/c2_tf32.json
python -c "
import json
for n in ('default','reference','c5_tf32','c2_tf32'):
    d=json.load(open('gpurun_out/final_c/%s.json'%n)); print(n, d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('clocks'))"
C3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_c/c3_launches.csv $C3 > gpurun_out/final_c/ncu_launch.log 2>&1
