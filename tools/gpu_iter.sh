# one build->measure iteration on the GPU box: tests, bench, ncu of level 10
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-iter}
python -m paper_2012_09739_b200.build > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -s -k "agreement or erfc_core" > gpurun_out/pytest_${TAG}_report.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_${TAG}.log
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum
timeout 300 python tools/profile_level.py > gpurun_out/prof_plain_${TAG}.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --metrics $M -k regex:level_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} python tools/profile_level.py > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_${TAG}.log; grep -E "Z ==|erfc" gpurun_out/pytest_${TAG}_report.log | head; tail -2 gpurun_out/bench_${TAG}.log | cut -c1-1500; tail -2 gpurun_out/ncu_${TAG}.log
