# image-only speculative blend: GPU tests + C3 bench over occupancy / unroll variants
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for v in base w5 u2 u2w5 p1 p1c6 u8 base; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 > gpurun_out/bench_$v.log 2>&1
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4), d['roofline']['kernel_ms_in_timed_region'])"
done
