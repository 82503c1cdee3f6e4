# the whole GPU suite on the bounds-checked build (-DLPMC_DEVICE_CHECKS:
# every table, shared-memory and output index checked on the device; a failed
# check prints the condition and traps the kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02_checks
LPMC_LIB=paper_2012_09739_b200/liblpmc_b200_checks.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_reference_tests.py > gpurun_out/r02_checks/pytest.log 2>&1; echo "checks exit $?" >> gpurun_out/r02_checks/pytest.log
grep -c "LPMC_DCHECK failed" gpurun_out/r02_checks/pytest.log; tail -6 gpurun_out/r02_checks/pytest.log
