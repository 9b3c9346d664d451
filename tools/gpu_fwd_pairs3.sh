# forward sub-block shape after the speculative blend: C3 sweep (image-only) and C2 iteration (tracking)
for v in base fp4 fp4u2 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C3 $(timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4))")"
done
for v in base tp2 base tp2; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C2 $(timeout 600 python tools/probe_train.py 300 2>&1 | tail -1)"
done
