# GPU box: the round's measurement artifacts -- default bench line, reference
# arm, smoke, ncu launch list of a short bench, ncu full capture of the top
# kernels (each ncu step only after its command exited 0 without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "exit $?" >> gpurun_out/bench_reference.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
timeout 300 python tools/profile_step.py > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"backward_quad|blend_forward|bin_front|ssim_bwd|ssim_fwd|chain_adam|preprocess" -c 7 \
    -o gpurun_out/full python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/bench_default.log | cut -c1-300; tail -2 gpurun_out/bench_reference.log | cut -c1-300
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/ncu_full.log
