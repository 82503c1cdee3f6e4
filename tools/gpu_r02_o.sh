cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o; mkdir -p $O
LPMC_LIB=paper_2012_09739_b200/liblpmc_b200_trace.so python tools/profile_level.py --level 12 --prec fp16 --payoff call --n 262144 --base $((12<<40)) --launches 1 > $O/trace_fp16.log 2>&1
grep -c "suspect path" $O/trace_fp16.log; grep "suspect path" $O/trace_fp16.log | head -12
