cd $GRAFT_REPO_ROOT
O=gpurun_out/r02cf; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "pow2" > $O/pytest_pow2.log 2>&1; echo "pytest exit $?" >> $O/pytest_pow2.log
tail -8 $O/pytest_pow2.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c5-l12-fp64 --level 12 --prec fp64 --n 4194304
t c5-l12-fp64k --level 12 --prec fp64 --kahan 1 --n 4194304
t c1-l6-fp64-hat --level 6 --prec fp64 --approx exact --legs hat --n 1048576 --base 0
t c1-l12-fp64-hat --level 12 --prec fp64 --approx exact --legs hat --n 4194304 --base 0
cat $O/timing.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
