# build, full GPU tests, bench and per-config throughput (one iteration)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-q}
python -m paper_2012_09739_b200.build > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench exit $?" >> gpurun_out/bench_${TAG}.err
timeout 900 python tools/bench_configs.py > gpurun_out/configs_${TAG}.json 2> gpurun_out/configs_${TAG}.err; echo "configs exit $?" >> gpurun_out/configs_${TAG}.err
tail -2 gpurun_out/pytest_${TAG}.log; tail -1 gpurun_out/bench_${TAG}.err; cut -c1-300 gpurun_out/bench_${TAG}.json; tail -1 gpurun_out/configs_${TAG}.err
