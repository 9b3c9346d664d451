# per-splat anchor check for the row recurrence: tests on the variant, C3 / C4 A/B
XG_LIB_VARIANT=rsc timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
for v in base rsc rscu2 base rsc rscu2; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4), 'C4', round(d['stress_c4']['value'],1))")"
done
