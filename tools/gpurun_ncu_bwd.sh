cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_sparse" -c 1 -o gpurun_out/sparse python tools/profile_step.py > gpurun_out/ncu_sparse.log 2>&1
PROF_STEPS=1 SS_BWD_WAVEFRONT=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_splat" -c 1 -o gpurun_out/wavefront python tools/profile_step.py > gpurun_out/ncu_wave.log 2>&1
tail -3 gpurun_out/ncu_sparse.log gpurun_out/ncu_wave.log
