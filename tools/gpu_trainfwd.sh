# training forward (xg_composite_fwd_train): GPU tests, C2 iteration
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do echo "C2 $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_np -s 30 -c 1 \
    -o gpurun_out/ncu_fwdtrain python tools/probe_train.py 40 > /dev/null 2>&1; echo "rc=$?"
