nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_bench.log | cut -c1-1500
