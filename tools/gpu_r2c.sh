# fused ranges + tile order; training forward pairs per lane (1 vs 2) inside the overlapped pair
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2c_pytest.log
timeout 300 python -m pytest tests/test_gpu_train_pair.py tests/test_gpu_trainer.py -q -x 2>&1 | tail -1
XG_LIB_VARIANT=lite2 timeout 300 python -m pytest tests/test_gpu_train_pair.py tests/test_gpu_trainer.py tests/test_gpu_fused_loss.py -q -x 2>&1 | tail -1
for v in "" lite2 "" lite2; do
  XG_LIB_VARIANT=$v timeout 300 python tools/probe_train.py 2000 88 1000 2>&1 | tail -1
done
