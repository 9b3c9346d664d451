nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_reference_fullsize.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for v in old new old new; do
  if [ $v = old ]; then export XG_LIB_VARIANT=old; else unset XG_LIB_VARIANT; fi
  timeout 300 python bench.py --no-train --no-c1 --no-c5 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], d['stress_c4']['value'], d['roofline']['frac'])"
done
