# trainer: forward queued before the binning counter read
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do echo "C2 $(timeout 300 python tools/probe_train.py 400 2>&1 | tail -1)"; done
