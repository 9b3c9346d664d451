# bench.py --collective p2p under torchrun x2 on ONE GPU (XG_BENCH_SHARE_GPU=1: ranks share the
# device and talk over gloo) - exercises the multi-rank paths (strong + weak
# C3 sharding, the C5 data-parallel training block); not a measurement
XG_BENCH_SHARE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --train-iters-per-step 100 --no-c4 --collective p2p > gpurun_out/r02_multirank_p2p.log 2> gpurun_out/r02_multirank_p2p.err
echo "rc=$?"; tail -c 1500 gpurun_out/r02_multirank_p2p.log; tail -5 gpurun_out/r02_multirank_p2p.err
