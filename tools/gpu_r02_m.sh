# native binary16 instance: its tests, then ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r02m}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_native_half.py -m gpu -q -p no:cacheprovider -x > $O/pytest_native.log 2>&1; echo "pytest exit $?" >> $O/pytest_native.log
tail -15 $O/pytest_native.log
bash tools/ncu_capture.sh c4_l12_fp16 $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
tail -3 gpurun_out/ncu/c4_l12_fp16.log
python -c "import json; d=json.load(open('gpurun_out/ncu/c4_l12_fp16.json')); print(d['kernel'], d['fp64_lane_ops_per_path_step'], d['warp_inst_per_path_step'], d['co_limits'])"
