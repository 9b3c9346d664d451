for np_ in 0 1; do for pr in 0 1; do
  echo -n "nonpersistent=$np_ binprio=$pr: "
  XG_BATCH_NONPERSISTENT=$np_ XG_BIN_PRIORITY=$pr timeout 300 python bench.py --no-train --no-c4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['e2e']['value'],1), round(r['frac'],3), round(r['kernel_ms_in_timed_region'],3))"
done; done
