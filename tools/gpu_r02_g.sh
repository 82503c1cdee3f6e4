# direct-table exact Gaussians: timing first, then the GPU test suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r02g}; mkdir -p $O
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
t c4-l12-fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
t c4-l11-fp16 --level 11 --prec fp16 --payoff call --n 4194304 --base $((11<<40))
t c2-l10-fp32 --level 10 --prec fp32 --n 4194304
t c2-l10-fp32k --level 10 --prec fp32 --kahan 1 --n 4194304
t c3-l8-half2-bar --level 8 --prec fp16-ieee --legs bar --n 16777216
t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
t c5-l14-fp32-bar --level 14 --prec fp32 --legs bar --n 4194304
t c1-l6-fp64-hat --level 6 --prec fp64 --approx exact --legs hat --n 1048576 --base 0
cat $O/timing.log
timeout 300 python tools/z_ratio.py > $O/z_ratio.log 2>&1; cat $O/z_ratio.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -30 $O/pytest_gpu.log
