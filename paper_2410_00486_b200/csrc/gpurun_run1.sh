cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 100 python profile_step.py > gpurun_out/plain.log 2>&1 && \
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "exit $?"
