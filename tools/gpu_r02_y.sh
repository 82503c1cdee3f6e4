# functional check of the multi-rank flow on the final kernels: one rank vs
# two and four ranks sharing the one GPU (gloo collectives on host tensors),
# the same 2^24 paths per level in total -> the same check moments, bitwise
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02y; mkdir -p $O
timeout 600 python bench.py --gpus 1 --steps 3 --warmup 3 --scaling strong --paths 16777216 --no-cpu-baseline --no-c2 > $O/n1.log 2>&1; echo "n1 exit $?"
for N in 2 4; do
LPMC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510+N)) bench.py --gpus $N --steps 3 --warmup 3 --scaling strong --paths 16777216 --no-cpu-baseline --no-c2 > $O/n$N.log 2>&1; echo "n$N exit $?"
done
for f in n1 n2 n4; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$f', d['n_gpus'], '%.4e'%d['value'], d['check'])"; done
