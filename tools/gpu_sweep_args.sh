# C3 sweep A/B over bench.py arguments (ARGS="--batch 16|--streams 6"), alternated with the default
IFS='|' read -ra alts <<< "$ARGS"
for rep in 1 2; do
  for a in "" "${alts[@]}"; do
    timeout 900 python bench.py --no-cpu-baseline --no-c5 --no-train --no-c1 --no-c4 $a > gpurun_out/sarg.log 2>&1
    echo -n "[$a] "; tail -1 gpurun_out/sarg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
