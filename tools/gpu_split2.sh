# split-half default: GPU tests, ncu of the batched launch
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/ncu_fwd_split python tools/prof_batch.py 3 > /dev/null 2>&1; echo "rc=$?"
