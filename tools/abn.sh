# A/B/... of kernel variants at two training phases (iterations 6-15 and
# 251-260): "base" = the tree as sent, then every tools/_ab_<name>/ directory
# (its .cu/.cuh files copied over csrc/ on top of the base sources).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abn
D=paper_2410_00486_b200/csrc
rm -rf /tmp/abn_base; mkdir -p /tmp/abn_base && cp $D/*.cu $D/*.cuh /tmp/abn_base/
make -s -C $D > /dev/null 2>&1
run() {
  PROF_WARM=5 timeout 200 python tools/profile_kernels.py > gpurun_out/abn/$1_early.txt 2>&1
  PROF_WARM=250 timeout 300 python tools/profile_kernels.py > gpurun_out/abn/$1_conv.txt 2>&1
}
run base
for d in tools/_ab_*/; do
  v=$(basename $d); v=${v#_ab_}
  cp /tmp/abn_base/* $D/
  cp $d/*.cu* $D/ 2>/dev/null
  make -s -C $D > gpurun_out/abn/${v}_build.txt 2>&1 || { echo "build $v failed"; cat gpurun_out/abn/${v}_build.txt | tail; continue; }
  run $v
done
cp /tmp/abn_base/* $D/ && make -s -C $D > /dev/null 2>&1
for ph in early conv; do for f in gpurun_out/abn/*_$ph.txt; do
  echo "== $(basename $f .txt)"; grep -v Warn $f | grep "us/step" | head -${AB_TOP:-3}; grep "per step" $f
done; done
