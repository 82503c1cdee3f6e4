cd $GRAFT_REPO_ROOT
for V in 4 3 2; do
  LPMC_NVCC_EXTRA="-DLPMC_GLIBC_MIN_CTAS=$V" python -m paper_2012_09739_b200.build --force > /dev/null 2>&1 || { echo "BUILD FAILED $V"; continue; }
  echo "ctas=$V l10 $(python tools/profile_level.py --time --exact-z glibc | tail -1) | c1 $(python tools/profile_level.py --time --exact-z glibc --legs hat --prec fp64 --approx exact --level 6 --n 1048576 | tail -1)"
done
