# lane-private tables: GPU tests, A/B against the round-1 kernels (base .so),
# one ncu capture of the C4 level-12 fp16 kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for rep in 1 2; do
for V in base lane; do
  LIB=paper_2012_09739_b200/liblpmc_b200.so; [ $V = base ] && LIB=paper_2012_09739_b200/liblpmc_b200_base.so
  echo "$V c4-l12-fp16 $(LPMC_LIB=$LIB timeout 300 python tools/profile_level.py --time --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40)) | tail -1)" >> $O/ab.log
  echo "$V c4-l12-fp32 $(LPMC_LIB=$LIB timeout 300 python tools/profile_level.py --time --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36)) | tail -1)" >> $O/ab.log
  echo "$V c2-l10-fp32 $(LPMC_LIB=$LIB timeout 300 python tools/profile_level.py --time --level 10 --prec fp32 --n 4194304 | tail -1)" >> $O/ab.log
done
done
bash tools/ncu_capture.sh c4_l12_fp16_lane $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
tail -3 $O/pytest_gpu.log; cat $O/ab.log; tail -40 gpurun_out/ncu/c4_l12_fp16_lane.md
