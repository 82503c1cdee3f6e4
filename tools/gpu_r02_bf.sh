cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bf; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_native_bf16.py -m gpu -q -p no:cacheprovider -x > $O/pytest_bf16.log 2>&1; echo "pytest exit $?" >> $O/pytest_bf16.log
tail -15 $O/pytest_bf16.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t l12-bf16 --level 12 --prec bf16 --n 4194304
t l12-bf16-kahan --level 12 --prec bf16 --kahan 1 --n 4194304
t l8-bf16-bar --level 8 --prec bf16 --legs bar --n 16777216
echo "l12-bf16-emulated $(LPMC_NO_NATIVE_BF16=1 timeout 300 python tools/profile_level.py --time --level 12 --prec bf16 --n 4194304 | tail -1)" >> $O/timing.log
echo "l8-bf16-bar-emulated $(LPMC_NO_NATIVE_BF16=1 timeout 300 python tools/profile_level.py --time --level 8 --prec bf16 --legs bar --n 16777216 | tail -1)" >> $O/timing.log
cat $O/timing.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
