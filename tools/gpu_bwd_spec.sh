# speculative reverse replay: GPU tests, C2 iteration timing A/B against XG_BWD_SPEC=0, ncu of the backward
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in spec nobspec spec nobspec; do
  if [ $v = spec ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo $v; timeout 600 python tools/probe_train.py 400 2>&1 | tail -1
done
unset XG_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd_ck -s 30 -c 1 \
    -o gpurun_out/ncu_bwd_train python tools/probe_train.py 40 > gpurun_out/ncu_bwd_train.log 2>&1; echo "rc=$?"
export XG_LIB_VARIANT=nobspec
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd_ck -s 30 -c 1 \
    -o gpurun_out/ncu_bwd_train_nospec python tools/probe_train.py 40 > gpurun_out/ncu_bwd_train.log 2>&1; echo "rc=$?"
