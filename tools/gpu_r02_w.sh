# Kahan on native binary16: its tests, timings, then the whole suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r02w}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_native_half.py -m gpu -q -p no:cacheprovider -x > $O/pytest_native.log 2>&1; echo "pytest exit $?" >> $O/pytest_native.log
tail -12 $O/pytest_native.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c3-l8-fp16-bar-kahan --level 8 --prec fp16 --legs bar --kahan 1 --n 16777216
t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
t c4-l12-fp16-kahan --level 12 --prec fp16 --payoff call --kahan 1 --n 4194304 --base $((12<<40))
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
echo "c4-l12-fp16-kahan-emulated $(LPMC_NO_NATIVE_HALF=1 timeout 300 python tools/profile_level.py --time --level 12 --prec fp16 --payoff call --kahan 1 --n 4194304 --base $((12<<40)) | tail -1)" >> $O/timing.log
cat $O/timing.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
