# backward reduction through shared memory: GPU tests, C2 iteration A/B, ncu of the backward
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in base noredsm base noredsm; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"
done
unset XG_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd_ck -s 30 -c 1 \
    -o gpurun_out/ncu_bwd_red python tools/probe_train.py 40 > /dev/null 2>&1; echo "rc=$?"
