# ncu captures of the persistent direct-table kernels (C4 level 12 fp16 / fp32)
cd $GRAFT_REPO_ROOT
bash tools/ncu_capture.sh c4_l12_fp16 $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
bash tools/ncu_capture.sh c4_l12_fp32 $((4194304 * 4096)) --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
tail -3 gpurun_out/ncu/c4_l12_fp16.log
for f in gpurun_out/ncu/*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['fp64_lane_ops_per_path_step'], d['warp_inst_per_path_step'], d['co_limits'])"; done
