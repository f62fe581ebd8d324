cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py tests/test_gpu_sanitizer.py -m gpu -q --timeout 300 -rf > gpurun_out/pytest_m.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_m.log
tail -4 gpurun_out/pytest_m.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config4 --no-e2e > gpurun_out/bench_m.log 2>&1
tail -1 gpurun_out/bench_m.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d.get('converged') or {}
print(round(d['value'],1), d['stage_ms'], 'conv', round(c.get('value',0),1), c.get('stage_ms'))"
