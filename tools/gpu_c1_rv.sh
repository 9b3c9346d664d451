for rv in 4 8; do
XG_RV_STREAMS=$rv timeout 300 python bench.py --no-c4 --no-train --no-c5 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['fwdbwd_c1']; print('rv $rv C1', round(c['value'],1), 'C1 e2e', round(c['e2e']['value'],1), 'C3', round(d['value'],1), 'C3 e2e', round(d['e2e']['value'],1), 'rv', round(d['e2e']['render_view_loop']['value'],1))"
done
