# sweep A/B of several tuning builds (VARIANTS="a b"), alternated with the default: C3 / C4 bench lines
for rep in 1 2; do for v in "" $VARIANTS; do
  XG_LIB_VARIANT=$v timeout 900 python bench.py --no-cpu-baseline --no-c5 --no-train --no-c1 > gpurun_out/sab.log 2>&1
  echo -n "[$v] "; tail -1 gpurun_out/sab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C4', round(d['stress_c4']['value'],1))"
done; done
