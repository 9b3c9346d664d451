# round-2 check: GPU tests, smoke, default bench (+ CPU baselines), reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 1500 python bench.py > gpurun_out/r2_bench.log 2>gpurun_out/r2_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r2_bench.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2_bench_ref.log | cut -c1-300
