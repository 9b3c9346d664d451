# C3 throughput vs views per compositing launch and binning streams
for b in 8 12 16; do
  timeout 300 python bench.py --no-train --no-c1 --no-c5 --no-c4 --no-cpu-baseline --steps 5 --warmup 3 --batch $b 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('batch $b', round(d['value'],1), round(d['e2e']['value'],1))"
done
