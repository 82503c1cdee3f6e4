# full evidence refresh on one GPU: tests, bench (default + reference arm),
# launch list, per-config throughput, callers bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r}
python -m paper_2012_09739_b200.build > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench exit $?" >> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref exit $?" >> gpurun_out/bench_ref_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch list exit $?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs_${TAG}.json 2> gpurun_out/configs_${TAG}.err; echo "configs exit $?" >> gpurun_out/configs_${TAG}.err
timeout 900 python tools/bench_callers.py > gpurun_out/callers_${TAG}.json 2> gpurun_out/callers_${TAG}.err; echo "callers exit $?" >> gpurun_out/callers_${TAG}.err
tail -1 gpurun_out/pytest_${TAG}.log; tail -1 gpurun_out/bench_${TAG}.err; cut -c1-400 gpurun_out/bench_${TAG}.json; tail -1 gpurun_out/bench_ref_${TAG}.err; cut -c1-300 gpurun_out/bench_ref_${TAG}.json; tail -1 gpurun_out/ncu_launch_${TAG}.log; tail -1 gpurun_out/configs_${TAG}.err; tail -1 gpurun_out/callers_${TAG}.err
