# lane tables + packed fp32 pairs: tests, A/B (base = round 1, flat = packed
# pairs on the flat table, main = both), Z error ratio, one ncu capture.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/z_ratio.py > $O/z_ratio.log 2>&1
P=paper_2012_09739_b200
for rep in 1 2; do
for V in base flat main; do
  LIB=$P/liblpmc_b200_$V.so; [ $V = main ] && LIB=$P/liblpmc_b200.so
  t() { echo "$V $1 $(LPMC_LIB=$LIB timeout 300 python tools/profile_level.py --time "${@:2}" | tail -1)" >> $O/ab.log; }
  t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
  t c4-l12-fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
  t c2-l10-fp32 --level 10 --prec fp32 --n 4194304
  t c2-l10-fp32k --level 10 --prec fp32 --kahan 1 --n 4194304
  t c3-l8-half2-bar --level 8 --prec fp16-ieee --legs bar --n 16777216
  t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
  t c5-l14-fp32-bar --level 14 --prec fp32 --legs bar --n 4194304
done
done
bash tools/ncu_capture.sh c4_l12_fp16_main $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
tail -15 $O/pytest_gpu.log; cat $O/z_ratio.log; cat $O/ab.log; grep -E "fp64 lane|warp-instructions per|issue_active|fp64_cycles" gpurun_out/ncu/c4_l12_fp16_main.md
