# power-of-two step folding: tests, timing, ncu demands -> bench, device
# bounds-check build over the GPU tests, functional 2-rank bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
t() { echo "$1 $(timeout 300 python tools/profile_level.py --time "${@:2}" | tail -1)" >> $O/timing.log; }
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
t c4-l12-fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
t c4-l11-fp16 --level 11 --prec fp16 --payoff call --n 4194304 --base $((11<<40))
t c2-l10-fp32 --level 10 --prec fp32 --n 4194304
t c2-l10-fp32k --level 10 --prec fp32 --kahan 1 --n 4194304
t c3-l8-fp16-bar --level 8 --prec fp16 --legs bar --n 16777216
t c5-l14-fp32-bar --level 14 --prec fp32 --legs bar --n 4194304
bash tools/ncu_capture.sh c4_l12_fp16 $((4194304 * 4096)) --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
bash tools/ncu_capture.sh c4_l12_fp32 $((4194304 * 4096)) --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
cp gpurun_out/ncu/c4_l12_fp16.json profiles/r02_c4_l12_demands.json
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c2 --scaling strong --paths 4194304 > $O/bench_n1_strong.log 2>&1
LPMC_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline --no-c2 --scaling strong --paths 4194304 > $O/bench_n2_shared.log 2>&1; echo "n2 exit $?" >> $O/bench_n2_shared.log
LPMC_LIB=paper_2012_09739_b200/liblpmc_b200_checks.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not reference_tests" > $O/pytest_checks.log 2>&1; echo "checks exit $?" >> $O/pytest_checks.log
tail -4 $O/pytest_gpu.log; cat $O/timing.log; tail -2 $O/bench.log | cut -c1-1200; tail -1 $O/bench_ref.log | cut -c1-300
python - <<'PY'
import json
for f in ["gpurun_out/r02e/bench_n1_strong.log", "gpurun_out/r02e/bench_n2_shared.log"]:
    try:
        line = [l for l in open(f) if l.startswith("{")][-1]
        print(f, json.loads(line)["check"])
    except Exception as e:
        print(f, "no line", e)
PY
tail -3 $O/pytest_checks.log
