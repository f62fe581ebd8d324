cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in Q U; do
  E=""; [ $v = U ] && E="SS_BWD_UNIT=1"
  env $E PROF_WARM=250 PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_" -c 1 -o gpurun_out/bq_$v python tools/profile_step.py > gpurun_out/ncu_bq_$v.log 2>&1
  tail -1 gpurun_out/ncu_bq_$v.log
done
