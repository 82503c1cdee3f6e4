# final measurement of the round-2 kernels: tests, per-precision timing and
# ncu captures, the C4 demands -> bench (the driver's own command lines),
# the reference arm, the launch list, the Z ratio.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${RUN:-r02final}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" | tail -1)" >> $O/timing.log; }
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
t c4-l12-fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
t c4-l11-fp16 --level 11 --prec fp16 --payoff call --n 4194304 --base $((11<<40))
t c2-l10-fp32 --level 10 --prec fp32 --n 4194304
t c2-l10-fp32k --level 10 --prec fp32 --kahan 1 --n 4194304
t c3-l8-half2-bar --level 8 --prec fp16-ieee --legs bar --n 16777216
t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
t c5-l14-fp32-bar --level 14 --prec fp32 --legs bar --n 4194304
t c1-l6-fp64-hat --level 6 --prec fp64 --approx exact --legs hat --n 1048576 --base 0
bash tools/ncu_capture.sh c4_l12_fp16 $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
cp gpurun_out/ncu/c4_l12_fp16.json profiles/r02_c4_l12_demands.json
bash tools/ncu_capture.sh c4_l12_fp32 $((4194304 * 4096)) --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
bash tools/ncu_capture.sh c3_l8_half2_bar $((16777216 * 256)) --level 8 --prec fp16-ieee --legs bar --n 16777216
bash tools/ncu_capture.sh c3_l8_fp16_bar $((16777216 * 256)) --level 8 --prec fp16 --legs bar --n 16777216
bash tools/ncu_capture.sh c5_l14_fp32_bar $((4194304 * 16384)) --level 14 --prec fp32 --legs bar --n 4194304
bash tools/ncu_capture.sh c2_l10_fp32 $((4194304 * 1024)) --level 10 --prec fp32 --n 4194304
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo "ref exit $?" >> $O/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c2 > $O/ncu_launch.log 2>&1; echo "ncu launches exit $?" >> $O/ncu_launch.log
timeout 300 python tools/z_ratio.py > $O/z_ratio.log 2>&1
tail -3 $O/pytest_gpu.log; cat $O/timing.log; tail -2 $O/bench.log | cut -c1-800; tail -2 $O/bench_ref.log | cut -c1-300; tail -1 $O/ncu_launch.log; cat $O/z_ratio.log
for f in gpurun_out/ncu/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['fp64_lane_ops_per_path_step'], d['warp_inst_per_path_step'], d['co_limits']['issue_active_pct'], d['co_limits']['fp64_pipe_active_pct'])"; done
# A/B: the fp32-carried emulation instead of native binary16 (same build)
echo "c4-l12-fp16-emulated $(LPMC_NO_NATIVE_HALF=1 timeout 300 python tools/profile_level.py --time --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40)) | tail -1)" >> $O/timing.log
echo "c4-l11-fp16-emulated $(LPMC_NO_NATIVE_HALF=1 timeout 300 python tools/profile_level.py --time --level 11 --prec fp16 --payoff call --n 4194304 --base $((11<<40)) | tail -1)" >> $O/timing.log
echo "c4-l12-fp16-glibc $(timeout 300 python tools/profile_level.py --time --level 12 --prec fp16 --payoff call --n 1048576 --base $((12<<40)) --exact-z glibc | tail -1)" >> $O/timing.log
tail -3 $O/timing.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c4-l12-fp16-kahan --level 12 --prec fp16 --payoff call --kahan 1 --n 4194304 --base $((12<<40))
t c3-l8-fp16-bar-kahan --level 8 --prec fp16 --legs bar --kahan 1 --n 16777216
t c5-l12-fp64 --level 12 --prec fp64 --n 4194304
t c5-l12-bf16 --level 12 --prec bf16 --n 4194304
t c5-l12-fp16ieee --level 12 --prec fp16-ieee --n 4194304
tail -5 $O/timing.log
