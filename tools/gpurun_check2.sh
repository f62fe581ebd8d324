cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -rf > gpurun_out/pytest_c2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_c2.log
tail -4 gpurun_out/pytest_c2.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d.get('converged') or {}
print(round(d['value'],1), d['gpu_launches'], d['stage_ms'], 'e2e', d['e2e']['value'], 'conv', round(c.get('value',0),1), c['e2e']['value'], 'cfg4', d['config4']['value'], d['config4']['gpu_launches'])"
