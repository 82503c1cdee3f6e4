# build + the GPU tests of the callers layer + the full GPU suite + callers bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-callers}
python -m paper_2012_09739_b200.build > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_callers.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_${TAG}_callers.log 2>&1; echo "callers exit $?" >> gpurun_out/pytest_${TAG}_callers.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 900 python tools/bench_callers.py > gpurun_out/callers_${TAG}.json 2> gpurun_out/callers_${TAG}.err; echo "bench_callers exit $?" >> gpurun_out/callers_${TAG}.err
tail -15 gpurun_out/pytest_${TAG}_callers.log; tail -3 gpurun_out/pytest_${TAG}.log; tail -3 gpurun_out/callers_${TAG}.err
