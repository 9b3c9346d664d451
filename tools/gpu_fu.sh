for v in base fu2 fu3 base fu2 fu3; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), 'C4', round(d['stress_c4']['value'],1))")"
done
