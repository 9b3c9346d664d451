# C3 binning chunk count at T = 1024: bin stage + sweep + C2
for v in base bs888 bs1776 bs222 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 300 python tools/probe.py 152 512 20 2>&1 | grep 'per view')"
  echo "$v C3 $(timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")"
  echo "$v C2 $(timeout 600 python tools/probe_train.py 300 2>&1 | tail -1)"
done
