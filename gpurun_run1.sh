cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 500 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_default.log
timeout 400 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.log 2>&1
echo "ref exit $?" >> gpurun_out/bench_reference.log
timeout 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 100 env PROF_STEPS=1 python profile_step.py > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"backward_splat|blend_forward" -c 2 -o gpurun_out/prof_r01_top env PROF_STEPS=1 python profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench_default.log | cut -c1-400; tail -2 gpurun_out/bench_reference.log | cut -c1-300
