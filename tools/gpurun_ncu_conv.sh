cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_WARM=250 timeout 300 python tools/profile_step.py > gpurun_out/plain_conv.log 2>&1 && \
PROF_WARM=250 PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_quad|blend_forward|bin_front|ssim_bwd|ssim_fwd|chain_adam|preprocess" -c 7 \
    -o gpurun_out/conv_full python tools/profile_step.py > gpurun_out/ncu_conv.log 2>&1
tail -2 gpurun_out/ncu_conv.log
