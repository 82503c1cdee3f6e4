# default build (flat tables, scalar bar legs): tests (incl. the reference's
# own unit tests + acceptance gate), Z ratio, the C4 bench, ncu captures of
# the C4 and per-precision kernels, the bench launch list, memcheck.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -m pytest tests/test_reference_tests.py -m gpu -q -s -p no:cacheprovider > $O/reftests.log 2>&1
timeout 300 python tools/z_ratio.py > $O/z_ratio.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
bash tools/ncu_capture.sh c4_l12_fp16 $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
bash tools/ncu_capture.sh c4_l12_fp32 $((4194304 * 4096)) --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
bash tools/ncu_capture.sh c3_l8_half2_bar $((16777216 * 256)) --level 8 --prec fp16-ieee --legs bar --n 16777216
bash tools/ncu_capture.sh c3_l8_fp16_bar $((16777216 * 256)) --level 8 --prec fp16 --legs bar --n 16777216
bash tools/ncu_capture.sh c5_l14_fp32_bar $((4194304 * 16384)) --level 14 --prec fp32 --legs bar --n 4194304
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c2 > $O/ncu_launch.log 2>&1; echo "ncu launches exit $?" >> $O/ncu_launch.log
timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize.py > $O/memcheck.log 2>&1; echo "memcheck exit $?" >> $O/memcheck.log
tail -6 $O/pytest_gpu.log; tail -25 $O/reftests.log; cat $O/z_ratio.log; tail -2 $O/bench.log | cut -c1-600; tail -1 $O/ncu_launch.log; tail -4 $O/memcheck.log
for f in gpurun_out/ncu/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['fp64_lane_ops_per_path_step'], d['warp_inst_per_path_step'], d['co_limits']['issue_active_pct'], d['co_limits']['fp64_pipe_active_pct'])"; done
