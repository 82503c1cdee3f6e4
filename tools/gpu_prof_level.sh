# ncu --set full capture of the C2 level-10 launch (after its plain run exits 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-prof}
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum
timeout 300 python tools/profile_level.py > gpurun_out/prof_plain_${TAG}.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --metrics $M -k regex:level_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} python tools/profile_level.py > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
