# refreshed caller and per-config benches on the final kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python tools/bench_callers.py > $O/callers.json 2> $O/callers.err; echo "callers exit $?"
timeout 1500 python tools/bench_configs.py > $O/configs.json 2> $O/configs.err; echo "configs exit $?"
tail -3 $O/callers.err; tail -3 $O/configs.err; head -c 1500 $O/callers.json
