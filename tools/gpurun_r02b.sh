cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
tail -20 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log | cut -c1-400
