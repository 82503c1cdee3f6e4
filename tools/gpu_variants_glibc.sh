# A/B of nvcc define variants on the glibc-mode level kernel (C2 level 10)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/variants_${1:-glibc}.log
: > $OUT
for V in ${VARIANTS}; do
  [ "$V" = "default" ] && V=""
  LPMC_NVCC_EXTRA="$(echo $V | tr ',' ' ')" python -m paper_2012_09739_b200.build --force > gpurun_out/build_variant.log 2>&1 || { echo "BUILD FAILED $V" >> $OUT; continue; }
  T=$(timeout 900 python -m pytest tests/test_gpu_glibc.py tests/test_veltkamp.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1)
  for K in 0 1; do
    echo "variant [$V] glibc kahan=$K $(python tools/profile_level.py --time --exact-z glibc --kahan $K | tail -1) | tests: $T" >> $OUT
  done
  echo "variant [$V] fast fp16 bar l8 $(python tools/profile_level.py --time --prec fp16 --legs bar --level 8 | tail -1)" >> $OUT
done
cat $OUT
