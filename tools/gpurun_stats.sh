cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_ITERS=6 timeout 300 python tools/bwd_stats.py > gpurun_out/bwd_stats2.jsonl 2>&1
PROF_ITERS=250 timeout 300 python tools/bwd_stats.py >> gpurun_out/bwd_stats2.jsonl 2>&1
cat gpurun_out/bwd_stats2.jsonl
