# views per compositing launch with the current kernels
for b in 12 10 15 12 10 15; do
  echo "batch $b $(timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 --batch $b 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4))")"
done
