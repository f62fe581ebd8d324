cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config4 > gpurun_out/bench.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
for f in bench; do tail -1 gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d.get('converged') or {}
print('$f', round(d['value'],1), d['stage_ms'].get('backward'), 'conv', round(c.get('value',0),1), (c.get('stage_ms') or {}).get('backward'), 'e2e', (d.get('e2e') or {}).get('value'))"; done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_sparse" -c 1 -o gpurun_out/sparse2 python tools/profile_step.py > gpurun_out/ncu_sparse.log 2>&1
tail -2 gpurun_out/ncu_sparse.log
