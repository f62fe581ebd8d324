cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
rm -f gpurun_out/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
tail -30 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-300
