cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k range -p no:cacheprovider > gpurun_out/pytest_range.log 2>&1
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum
timeout 300 python tools/profile_level.py > gpurun_out/prof_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --metrics $M -k regex:level_kernel -s 1 -c 1 -o gpurun_out/prof_l10_fp32 python tools/profile_level.py > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/pytest_range.log; tail -2 gpurun_out/bench.log | cut -c1-2500; tail -3 gpurun_out/ncu_full.log; tail -2 gpurun_out/ncu_launch.log
