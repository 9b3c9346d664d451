# preprocess / preprocess-backward occupancy variants
for v in base pre12 pre16 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1))") $(timeout 300 python tools/probe.py 152 512 20 2>&1 | grep 'per view' | cut -c1-40)"
done
for v in base pb5 pb8 base pb5; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C2 $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"
done
