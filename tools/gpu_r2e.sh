# one memset for both balanced-path scans: GPU tests, C2 iteration times
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2e_pytest.log
for i in 1 2 3; do timeout 300 python tools/probe_train.py 2000 88 1000 2>&1 | tail -1; done
