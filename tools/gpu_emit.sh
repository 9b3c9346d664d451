# bin emit owner lookup: GPU tests, C3 / C4 bin stage, C3 sweep
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in base bt128 base bt128; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v C3 $(timeout 300 python tools/probe.py 152 512 20 2>&1 | grep 'per view')"
  echo "$v C4 $(timeout 300 python tools/probe.py 196 1024 8 2>&1 | grep 'per view')"
done
unset XG_LIB_VARIANT
timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4), 'C4', round(d['stress_c4']['value'],1))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4e.csv python tools/prof_c3.py 1 196 1024 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c4e.csv 2>/dev/null | grep -i "bin_\|os_pass"
