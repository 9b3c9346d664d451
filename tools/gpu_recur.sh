# multiplicative row recurrence: GPU tests, C3 / C4 A/B, ncu of the batched launch
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in base norecur base norecur; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms_in_timed_region'],3), 'C4', round(d['stress_c4']['value'],1))")"
done
unset XG_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/ncu_fwd_recur python tools/prof_batch.py 3 > /dev/null 2>&1; echo "rc=$?"
