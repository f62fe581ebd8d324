cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python debug_stages.py > gpurun_out/debug.log 2>&1
echo "debug exit $?" >> gpurun_out/debug.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
tail -30 gpurun_out/debug.log; tail -5 gpurun_out/bench.log
