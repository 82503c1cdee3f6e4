cd $GRAFT_REPO_ROOT
O=gpurun_out/r02z; mkdir -p $O
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c5-l12-fp64 --level 12 --prec fp64 --n 4194304
t c5-l12-fp64k --level 12 --prec fp64 --kahan 1 --n 4194304
t c5-l11-fp64 --level 11 --prec fp64 --n 4194304
t c5-l12-fp32 --level 12 --prec fp32 --n 4194304
t c5-l11-fp32 --level 11 --prec fp32 --n 4194304
t c5-l12-bf16 --level 12 --prec bf16 --n 4194304
t c5-l12-fp16ieee --level 12 --prec fp16-ieee --n 4194304
t c5-l12-fp16ieee-k --level 12 --prec fp16-ieee --kahan 1 --n 4194304
cat $O/timing.log
