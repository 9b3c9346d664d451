# multi-rank code path on ONE GPU (gloo, ranks share the device): not a measurement
set -x
XG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mr.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/mr.log | cut -c1-600
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.log 2>&1; echo "ref rc=$?"
tail -2 gpurun_out/mr_ref.log | cut -c1-300
