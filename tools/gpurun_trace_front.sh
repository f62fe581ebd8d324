cd $GRAFT_REPO_ROOT
make -s -C paper_2410_00486_b200/csrc clean
make -s -C paper_2410_00486_b200/csrc EXTRA=-DSS_FE_TRACE -j8 > /dev/null 2>&1
python tools/trace_front.py > gpurun_out/trace_front.txt 2>&1
cat gpurun_out/trace_front.txt
