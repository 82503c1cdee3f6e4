# time the C2 level-10 launch for several nvcc define variants (experiments);
# each variant also runs the bit-exact path / moment parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/variants_${1:-x}.log
: > $OUT
for V in ${VARIANTS}; do
  [ "$V" = "default" ] && V=""
  LPMC_NVCC_EXTRA="$(echo $V | tr ',' ' ')" python -m paper_2012_09739_b200.build --force > gpurun_out/build_variant.log 2>&1 || { echo "BUILD FAILED $V" >> $OUT; continue; }
  T=$(timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_callers.py -m gpu -q -p no:cacheprovider -k "paths_vs_reference or moments or two_way_paths or legs_and_payoff or fallback" 2>&1 | tail -1)
  for K in 0 1; do
    echo "variant [$V] kahan=$K $(python tools/profile_level.py --time --kahan $K | tail -1) | tests: $T" >> $OUT
  done
done
cat $OUT
