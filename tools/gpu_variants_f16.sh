# A/B of nvcc define variants on the emulated fp16 (m = 10) legs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/variants_${1:-f16}.log
: > $OUT
for V in ${VARIANTS}; do
  [ "$V" = "default" ] && V=""
  LPMC_NVCC_EXTRA="$(echo $V | tr ',' ' ')" python -m paper_2012_09739_b200.build --force > gpurun_out/build_variant.log 2>&1 || { echo "BUILD FAILED $V" >> $OUT; continue; }
  T=$(timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1)
  for L in "all 10" "bar 8"; do set -- $L; for K in 0 1; do
    echo "variant [$V] fp16 legs=$1 level=$2 kahan=$K $(python tools/profile_level.py --time --prec fp16 --legs $1 --level $2 --kahan $K | tail -1) | tests: $T" >> $OUT
  done; done
done
cat $OUT
