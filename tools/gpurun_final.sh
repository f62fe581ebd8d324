# GPU box: the round's evidence -- full GPU suite with the full-size parity
# report, default bench line, reference arm, smoke, configs, backward work
# stats, API timing, sparse-backward ablation line, ncu launch list of a short
# bench, ncu full captures of the top kernels (iterations 6-25 and 251-270).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
nproc > $O/host.txt; lscpu | grep -i "model name" >> $O/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> $O/host.txt 2>&1
rm -f $O/parity_fullsize.jsonl
SS_PARITY_REPORT=$PWD/$O/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "exit $?" >> $O/bench_default.log
timeout 600 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "exit $?" >> $O/bench_reference.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 900 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
PROF_ITERS=6 timeout 300 python tools/bwd_stats.py > $O/bwd_stats.jsonl 2>&1
PROF_ITERS=250 timeout 300 python tools/bwd_stats.py >> $O/bwd_stats.jsonl 2>&1
timeout 300 python tools/api_timing.py > $O/api_timing.txt 2>&1
SS_BWD_SPARSE=1 timeout 600 python bench.py --no-cpu-baseline --no-config4 > $O/bench_sparse.log 2>&1
SS_BWD_UNIT=1 timeout 600 python bench.py --no-cpu-baseline --no-config4 > $O/bench_unit_chains.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-converged --no-config4 --no-e2e > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-converged --no-config4 --no-e2e \
    > $O/ncu_launches.log 2>&1
timeout 300 python tools/profile_step.py > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_quad|blend_forward|bin_front|ssim_bwd|ssim_fwd|chain_adam|preprocess" -c 7 \
    -o $O/full python tools/profile_step.py > $O/ncu_full.log 2>&1
PROF_WARM=250 PROF_STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_quad|blend_forward|bin_front|ssim_bwd|ssim_fwd|chain_adam|preprocess" -c 7 \
    -o $O/conv_full python tools/profile_step.py > $O/ncu_conv.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/bench_default.log | cut -c1-300; tail -2 $O/bench_reference.log | cut -c1-300; tail -2 $O/smoke.log
