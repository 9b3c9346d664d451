# GPU tests + C2 training launch list (per-kernel share of an iteration)
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/probe_train.py 300 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_train.csv python tools/probe_train.py 10 > /dev/null 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/launches_train.csv | head -14
