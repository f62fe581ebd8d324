# ncu --set full of the splat-wise backward at iteration 6 (early) and 251
# (converged) of the bench workload -> gpurun_out/bq_{early,conv}.ncu-rep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 5 250; do
  tag=early; [ $w = 250 ] && tag=conv
  PROF_WARM=$w PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_" -c 1 -o gpurun_out/bq_$tag python tools/profile_step.py > gpurun_out/ncu_bq_$tag.log 2>&1
  tail -1 gpurun_out/ncu_bq_$tag.log
done
