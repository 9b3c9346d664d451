# reverse-replay chunk size after the speculative backward: C2 iteration
XG_LIB_VARIANT=rc128 timeout 600 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
for v in base rc128 rc512 base rc128 rc512; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C2 $(timeout 300 python tools/probe_train.py 400 2>&1 | tail -1)"
done
