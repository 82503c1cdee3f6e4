# ncu --set full of one level launch on the GPU box, summarised there (the
# .ncu-rep files are too big to bring back): NAME PATH_STEPS profile_level args...
#   -> gpurun_out/ncu/NAME.{md,json,raw.csv,log}
# Runs the plain command first; captures only if it exited 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
N=$1; PS=$2; shift 2
D=gpurun_out/ncu
timeout 300 python tools/profile_level.py "$@" > $D/$N.plain.log 2>&1 || { echo "plain run failed" >> $D/$N.plain.log; exit 1; }
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_hadd_pred_on.sum,sm__sass_thread_inst_executed_op_hmul_pred_on.sum,sm__sass_thread_inst_executed_op_hfma_pred_on.sum,sm__sass_thread_inst_executed_op_integer_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fp16.sum
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:level_kernel -s 1 -c 1 -o /tmp/$N python tools/profile_level.py "$@" > $D/$N.log 2>&1
echo "ncu exit $?" >> $D/$N.log
ncu -i /tmp/$N.ncu-rep --page raw --csv > $D/$N.raw.csv 2>/dev/null
python tools/summarize_ncu.py full /tmp/$N.ncu-rep $PS > $D/$N.md 2>&1
python tools/summarize_ncu.py demands /tmp/$N.ncu-rep $PS "profile_level.py $*" > $D/$N.json 2>&1
ncu -i /tmp/$N.ncu-rep --page details > $D/$N.details.txt 2>&1
ncu -i /tmp/$N.ncu-rep --page source --csv --print-source sass > $D/$N.source.csv 2>/dev/null
rm -f /tmp/$N.ncu-rep
