# round-2 late check: the workspace mapping entry point (asot_map_to_anchors_ws) on one B200 --
# the mapping / edge / distributed GPU tests, then the default bench line (outputs under gpurun_out/final_b/)
mkdir -p gpurun_out/final_b
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_parity_full.py tests/test_gpu_bench_contract.py -m gpu -q -p no:cacheprovider -k "mapping or map_ws or nccl or dist or status or bench" > gpurun_out/final_b/gputest_map.log 2>&1; tail -3 gpurun_out/final_b/gputest_map.log
python bench.py > gpurun_out/final_b/bench_default.log 2>&1; tail -1 gpurun_out/final_b/bench_default.log > gpurun_out/final_b/bench_default.json
python -c "import json; d=json.load(open('gpurun_out/final_b/bench_default.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
