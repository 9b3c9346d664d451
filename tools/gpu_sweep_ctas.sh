for c in 5 4 3; do for ns in 4 6; do
  echo -n "fwd ctas/sm=$c streams=$ns: "
  XG_FWD_CTAS_PER_SM=$c timeout 300 python bench.py --no-train --no-c4 --no-cpu-baseline --streams $ns 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['kernel_ms_in_timed_region'],4))"
done; done
