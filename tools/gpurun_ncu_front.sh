# ncu --set full (with source) of the binning front end at iteration 6 of
# the bench workload -> gpurun_out/fe_early.ncu-rep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_WARM=5 PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"bin_front" -c 1 -o gpurun_out/fe_early python tools/profile_step.py > gpurun_out/ncu_fe.log 2>&1
tail -1 gpurun_out/ncu_fe.log
