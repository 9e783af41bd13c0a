# round-2 final: the GPU suite and smoke() on one B200 (outputs under gpurun_out/final/)
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/gputest.log 2>&1; tail -3 gpurun_out/final/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
