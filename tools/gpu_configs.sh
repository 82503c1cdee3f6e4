cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2012_09739_b200.build > gpurun_out/build_cfg.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_cfg.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_cfg.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo "configs exit $?"
tail -3 gpurun_out/pytest_cfg.log; tail -5 gpurun_out/configs.err
