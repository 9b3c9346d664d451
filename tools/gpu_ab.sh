# A/B of tuning builds (tools: _build.build_variant) against the default build:
#   VARIANTS="a b" bash tools/gpu_ab.sh   (each name loads csrc/_variants/libxgauss_<name>.so; "new" = default)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
VARIANTS=${VARIANTS:-"old new"}
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = new ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  g=$(timeout 100 python tools/probe_bin_graph.py 24 2>/dev/null | tail -1 | awk '{print $(NF)}')
  timeout 300 python bench.py --no-train --no-c1 --no-c5 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'bin', '$g', 'C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C4', round(d['stress_c4']['value'],1))"
done
done
