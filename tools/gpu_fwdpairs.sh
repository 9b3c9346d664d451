# forward pixel-pairs-per-lane variants: C3 sweep (bench, no CPU/C2/C4 blocks) and C2 training
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in "" f2 f4; do echo "== variant [$v]"; XG_LIB_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-train --no-c4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline'])"; done
for v in "" t2; do echo "== variant [$v]"; XG_LIB_VARIANT=$v timeout 300 python tools/probe_train.py 300 2>&1 | tail -1; done
