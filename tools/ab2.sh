# A/B of kernel variants at two training phases (iterations 6-15 and 251-260):
# A = the tree as sent, B = the tree with tools/_ab/ files over csrc/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A B; do
  if [ $v = B ]; then
    for f in tools/_ab/*.cu tools/_ab/*.cuh; do [ -f "$f" ] && cp "$f" paper_2410_00486_b200/csrc/; done
    make -s -C paper_2410_00486_b200/csrc > gpurun_out/ab_build.txt 2>&1 || { cat gpurun_out/ab_build.txt; exit 1; }
  fi
  PROF_WARM=5 timeout 200 python tools/profile_kernels.py > gpurun_out/ab2_${v}_early.txt 2>&1
  PROF_WARM=250 timeout 300 python tools/profile_kernels.py > gpurun_out/ab2_${v}_conv.txt 2>&1
done
for ph in early conv; do for v in A B; do
  echo "== $v $ph"; grep -v Warn gpurun_out/ab2_${v}_$ph.txt | grep "us/step" | head -${AB_TOP:-6}; grep "per step" gpurun_out/ab2_${v}_$ph.txt
done; done
