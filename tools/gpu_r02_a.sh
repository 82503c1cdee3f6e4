# Round 2, first GPU call: tests, the C4 bench, the reference arm, the ncu
# launch list and --set full captures of the C4 level-12 kernels and the
# per-precision kernels (each only after its plain command exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi -L > $O/smi.txt 2>&1; nproc >> $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref exit $?" >> $O/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c2 > $O/ncu_launch.log 2>&1; echo "ncu launches exit $?" >> $O/ncu_launch.log
prof() {  # name, args...
  local n=$1; shift
  timeout 300 python tools/profile_level.py "$@" > $O/$n.plain.log 2>&1 || { echo "plain failed" >> $O/$n.plain.log; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_kernel -s 1 -c 1 -o $O/$n python tools/profile_level.py "$@" > $O/$n.ncu.log 2>&1; echo "ncu exit $?" >> $O/$n.ncu.log
}
prof c4_l12_fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
prof c4_l12_fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
prof c3_l8_half2_bar --level 8 --prec fp16-ieee --legs bar --n 16777216
prof c5_l14_fp32_bar --level 14 --prec fp32 --legs bar --n 4194304
tail -3 $O/pytest_gpu.log; tail -2 $O/bench.log | cut -c1-4000; tail -2 $O/bench_ref.log | cut -c1-1500; tail -1 $O/ncu_launch.log; tail -n1 $O/*.ncu.log
