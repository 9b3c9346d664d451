for pc in 0; do for ns in ${NS:-2 3 4}; do
  echo -n "prio=$pc streams=$ns: "
  XG_PRIORITY_COMPOSITE=$pc timeout 300 python bench.py --no-train --no-c4 --no-cpu-baseline --streams $ns 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['kernel_ms_in_timed_region'],4))"
done; done
