# speculative tracking forward: GPU tests, C2 iteration timing A/B against XG_FWD_SPEC_TRACK=0, ncu of the backward
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in spec nost spec nost; do
  if [ $v = spec ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo $v; timeout 600 python tools/probe_train.py 400 2>&1 | tail -1
done
unset XG_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_np -s 30 -c 1 \
    -o gpurun_out/ncu_fwdtr_train python tools/probe_train.py 40 > gpurun_out/ncu_fwdtr_train.log 2>&1; echo "rc=$?"
export XG_LIB_VARIANT=nost
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_np -s 30 -c 1 \
    -o gpurun_out/ncu_fwdtr_train_nospec python tools/probe_train.py 40 > gpurun_out/ncu_fwdtr_train.log 2>&1; echo "rc=$?"
