# A/B of kernel variants through bench.py (device it/s at iterations 6-25
# and 251-270), alternating base and every tools/_ab_<name>/ overlay
# AB_ROUNDS times; prints one line per run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abb
D=paper_2410_00486_b200/csrc
mkdir -p /tmp/abb_base && cp $D/*.cu $D/*.cuh /tmp/abb_base/
rm -rf /tmp/abb_lib; mkdir -p /tmp/abb_lib
make -s -C $D > /dev/null 2>&1 && cp paper_2410_00486_b200/libss_b200.so /tmp/abb_lib/base.so
for d in tools/_ab_*/; do
  v=$(basename $d); v=${v#_ab_}
  cp /tmp/abb_base/* $D/; cp $d/*.cu* $D/ 2>/dev/null
  make -s -C $D > gpurun_out/abb/${v}_build.txt 2>&1 && cp paper_2410_00486_b200/libss_b200.so /tmp/abb_lib/$v.so
done
cp /tmp/abb_base/* $D/
b() {
  cp /tmp/abb_lib/$1.so paper_2410_00486_b200/libss_b200.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-config4 --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['converged']['value'],1))"
}
for i in $(seq ${AB_ROUNDS:-3}); do
  for f in /tmp/abb_lib/*.so; do b $(basename $f .so); done
done
cp /tmp/abb_lib/base.so paper_2410_00486_b200/libss_b200.so
