# A/B of the exact Gaussian's initial guess: fp32 x0 + Halley (default) vs Acklam (-DLPMC_X0_ACKLAM)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/ab_x0.log
: > $OUT
python -m paper_2012_09739_b200.build --force > gpurun_out/build_ab.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build_ab.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ab.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -s -k "agreement" > gpurun_out/agree_ab.log 2>&1
for K in 0 1; do echo "new kahan=$K $(python tools/profile_level.py --time --kahan $K | tail -1)" >> $OUT; done
LPMC_NVCC_EXTRA="-DLPMC_X0_ACKLAM" python -m paper_2012_09739_b200.build --force > gpurun_out/build_ab2.log 2>&1
for K in 0 1; do echo "acklam kahan=$K $(python tools/profile_level.py --time --kahan $K | tail -1)" >> $OUT; done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -s -k "agreement" > gpurun_out/agree_ab_acklam.log 2>&1
tail -3 gpurun_out/pytest_ab.log; cat $OUT; grep -iE "bitwise|agree|ulp" gpurun_out/agree_ab.log | head -5; grep -iE "bitwise|agree|ulp" gpurun_out/agree_ab_acklam.log | head -5
