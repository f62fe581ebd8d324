# ncu --set full of the kernels matching $K (regex), one launch each, at
# iteration PROF_WARM (default 5) of the bench workload -> gpurun_out/k_<tag>.ncu-rep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_WARM=${PROF_WARM:-5} PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  --profile-from-start off -k regex:"$K" -c ${NK:-6} -o gpurun_out/k_${TAG:-x} python tools/profile_step.py \
  > gpurun_out/ncu_k_${TAG:-x}.log 2>&1
tail -1 gpurun_out/ncu_k_${TAG:-x}.log
