# 2-pair forward: occupancy / unroll variants at C3 (bench, no CPU/C2/C4 blocks)
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in "" w5 w5u2 u2 w5u8 ""; do echo "== variant [$v]"; XG_LIB_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-train --no-c4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value'],1), round(d['e2e']['value'],1), round(r['frac'],4), round(r['kernel_ms_in_timed_region'],4))"; done
