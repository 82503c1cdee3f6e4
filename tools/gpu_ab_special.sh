cd $GRAFT_REPO_ROOT
VARIANTS="-DLPMC_EXACT_SPECIAL default" bash tools/gpu_variants.sh special
VARIANTS="-DLPMC_EXACT_SPECIAL default" bash tools/gpu_ncu_variants.sh special | grep "inst_executed.sum\|time_dur\|issue_active"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_special.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_special.log
tail -2 gpurun_out/pytest_special.log
