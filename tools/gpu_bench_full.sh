# round-end style: full bench (our arm) + reference arm, both N=1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.log
