cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python debug_stages.py > gpurun_out/debug.log 2>&1
echo "debug exit $?" >> gpurun_out/debug.log
tail -4 gpurun_out/debug.log
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 100 python profile_step.py > gpurun_out/plain.log 2>&1 && \
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python profile_step.py > gpurun_out/ncu_launch.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log
