# A/B of kernel variants on the GPU box: A = the tree as sent, B = the tree
# with every file under tools/_ab/ copied over its namesake in csrc/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
reps=${AB_REPS:-2}
for r in $(seq $reps); do
  timeout 200 python tools/profile_kernels.py > gpurun_out/ab_A_$r.txt 2>&1
done
for f in tools/_ab/*.cu tools/_ab/*.cuh; do [ -f "$f" ] && cp "$f" paper_2410_00486_b200/csrc/; done
make -s -C paper_2410_00486_b200/csrc > gpurun_out/ab_build.txt 2>&1 || { cat gpurun_out/ab_build.txt; exit 1; }
for r in $(seq $reps); do
  timeout 200 python tools/profile_kernels.py > gpurun_out/ab_B_$r.txt 2>&1
done
for r in $(seq $reps); do
  echo "== A run $r"; grep -v Warn gpurun_out/ab_A_$r.txt | grep "us/step" | head -${AB_TOP:-8}; grep "per step" gpurun_out/ab_A_$r.txt
  echo "== B run $r"; grep -v Warn gpurun_out/ab_B_$r.txt | grep "us/step" | head -${AB_TOP:-8}; grep "per step" gpurun_out/ab_B_$r.txt
done
