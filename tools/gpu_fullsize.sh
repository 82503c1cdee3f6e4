cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --durations=8 > gpurun_out/fullsize.log 2>&1; echo "pytest exit $?" >> gpurun_out/fullsize.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun1.log 2>&1; echo "torchrun exit $?" >> gpurun_out/torchrun1.log
tail -30 gpurun_out/fullsize.log; tail -3 gpurun_out/torchrun1.log | cut -c1-600
