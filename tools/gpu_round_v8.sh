# round check of HEAD: GPU tests, smoke, bench (+ reference arm), launch list of the bench, ncu of the batched compositing + backward
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-1500
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-train --no-c4 > gpurun_out/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/ncu_fwd_batch python tools/prof_batch.py 3 > gpurun_out/ncu_fwd_batch.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd -s 2 -c 1 \
    -o gpurun_out/ncu_bwd python tools/prof_c3.py 3 > gpurun_out/ncu_bwd.log 2>&1; echo "rc=$?"
