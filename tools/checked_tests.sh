# compute-sanitizer is closed on this pool: run the GPU suite on a build with device-side bounds
# checks instead (ASOT_CHECKED=1: every ASOT_DEV_CHECK traps with its file:line), then restore the
# product build.  Outputs under gpurun_out/checked/.
mkdir -p gpurun_out/checked
ASOT_CHECKED=1 python -m paper_2310_16123_b200._build > gpurun_out/checked/build.log 2>&1 && echo "checked build ok"
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked/gputest.log 2>&1; tail -3 gpurun_out/checked/gputest.log
grep -c "ASOT_CHECKED" gpurun_out/checked/gputest.log
python -m paper_2310_16123_b200._build > /dev/null 2>&1 && echo "product build restored"
