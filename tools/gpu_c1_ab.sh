# C1 fwd+bwd throughput vs views in flight and issue order (XG_C1_STREAMS, XG_C1_WAVE)
for cfg in "4 0" "4 1" "8 1" "16 1" "8 0"; do
  set -- $cfg
  XG_C1_STREAMS=$1 XG_C1_WAVE=$2 timeout 300 python bench.py --no-c4 --no-train --no-c5 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['fwdbwd_c1']; print('streams $1 wave $2', round(c['value'],1), 'e2e', round(c['e2e']['value'],1), 'C3', round(d['value'],1))"
done
