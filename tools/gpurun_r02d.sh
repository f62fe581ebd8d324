cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
PROF_ITERS=6 timeout 300 python tools/bwd_stats.py > gpurun_out/bwd_stats.jsonl 2>&1
PROF_ITERS=250 timeout 300 python tools/bwd_stats.py >> gpurun_out/bwd_stats.jsonl 2>&1
tail -8 gpurun_out/pytest_gpu.log; cat gpurun_out/bwd_stats.jsonl
