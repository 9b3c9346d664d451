# split-half image-only units: GPU tests on the variant build, C3 / C4 A/B
XG_LIB_VARIANT=split timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_split.log 2>&1; echo "pytest(split) rc=$?"; tail -2 gpurun_out/pytest_split.log
for v in base split splitu2 base split splitu2; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms_in_timed_region'],3), 'C4', round(d['stress_c4']['value'],1))")"
done
