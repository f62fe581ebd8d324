cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SS_BWD_SPARSE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py -m gpu -q --timeout 300 -rf -x > gpurun_out/pytest_sparse.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sparse.log
tail -3 gpurun_out/pytest_sparse.log
SS_BWD_SPARSE=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config4 --no-e2e > gpurun_out/bench_sparse.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config4 --no-e2e > gpurun_out/bench_wave.log 2>&1
for f in bench_sparse bench_wave; do tail -1 gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d.get('converged') or {}
print('$f', round(d['value'],1), d['stage_ms'].get('backward'), 'conv', round(c.get('value',0),1), (c.get('stage_ms') or {}).get('backward'))"; done
SS_BWD_SPARSE=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_sparse" -c 1 -o gpurun_out/sparse3 python tools/profile_step.py > gpurun_out/ncu_sparse.log 2>&1
tail -1 gpurun_out/ncu_sparse.log
