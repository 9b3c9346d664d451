# speculative image-only blend: GPU tests, then C3 bench A/B against the XG_FWD_SPEC=0 build
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for v in spec nospec spec; do
  if [ $v = spec ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 > gpurun_out/bench_$v.log 2>&1; echo "$v rc=$?"
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_ms_in_timed_region'])"
done
unset XG_LIB_VARIANT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/ncu_fwd_spec python tools/prof_batch.py 3 > gpurun_out/ncu_fwd_spec.log 2>&1; echo "rc=$?"
