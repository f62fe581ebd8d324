# A/B of an environment switch at two training phases (iterations 6-15 and
# 251-260): A = default, B = with $AB_ENV (e.g. AB_ENV=SS_BWD_UNIT=1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A B; do
  E=""; [ $v = B ] && E="$AB_ENV"
  env $E PROF_WARM=5 timeout 200 python tools/profile_kernels.py > gpurun_out/abe_${v}_early.txt 2>&1
  env $E PROF_WARM=250 timeout 300 python tools/profile_kernels.py > gpurun_out/abe_${v}_conv.txt 2>&1
done
for ph in early conv; do for v in A B; do
  echo "== $v $ph"; grep -v Warn gpurun_out/abe_${v}_$ph.txt | grep "us/step" | head -${AB_TOP:-6}; grep "per step" gpurun_out/abe_${v}_$ph.txt
done; done
