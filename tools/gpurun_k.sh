cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -rf /tmp/rt && cp -r $GRAFT_REPO_ROOT /tmp/rt && cd /tmp/rt/paper_2410_00486_b200/csrc && make -s clean && \
make -s -j8 FLAGS="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DSS_FE_TRACE" > /dev/null 2>&1
cd /tmp/rt && timeout 300 python tools/trace_front.py > $GRAFT_REPO_ROOT/gpurun_out/trace_front.txt 2>&1
PROF_ITERS=0 cd /tmp/rt && cat $GRAFT_REPO_ROOT/gpurun_out/trace_front.txt
