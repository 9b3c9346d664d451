# onesweep tile size (keys per CTA = 256 x rounds): C2 iteration, C3 sweep
for v in base osr4 osr2 base osr4; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C2 $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"
  echo "$v C3 $(timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")"
done
