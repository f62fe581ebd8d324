cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_guard.py -m gpu -q --timeout 300 -rf > gpurun_out/pytest_n.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_n.log
tail -4 gpurun_out/pytest_n.log
timeout 300 python tools/api_timing.py > gpurun_out/api_timing_n.txt 2>&1
grep "API path" gpurun_out/api_timing_n.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
