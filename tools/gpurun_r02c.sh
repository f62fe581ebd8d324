cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
echo "configs exit $?" >> gpurun_out/configs.err
timeout 300 python tools/profile_kernels.py > gpurun_out/kernels.txt 2>&1
tail -8 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/configs.jsonl; tail -3 gpurun_out/configs.err; grep -v Warn gpurun_out/kernels.txt | head -30
