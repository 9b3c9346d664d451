# onesweep windowed look-back: GPU tests, per-stage bin time / C3 sweep / C2 iteration per window size
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in base lb1 lb4 lb16 base lb1; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "== $v"
  timeout 300 python tools/probe.py 152 512 20 2>&1 | grep "per view"
  timeout 300 python tools/probe.py 196 1024 8 2>&1 | grep "per view"
  timeout 600 python bench.py --no-cpu-baseline --no-train --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4))"
  timeout 600 python tools/probe_train.py 300 2>&1 | tail -1
done
unset XG_LIB_VARIANT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_c3.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv 2>/dev/null | head -12
