cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r02p}; mkdir -p $O
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
t c4-l11-fp16 --level 11 --prec fp16 --payoff call --n 4194304 --base $((11<<40))
t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
cat $O/timing.log
timeout 1200 python -m pytest tests/test_gpu_native_half.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
tail -5 $O/pytest.log
