# middle-anchored row recurrence: GPU tests, path stats, C3 / C4 sweep
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
XG_LIB_VARIANT=bstats timeout 300 python tools/probe_fwd_stats.py 2>&1 | tail -2
for i in 1 2; do
echo "$(timeout 600 python bench.py --no-cpu-baseline --no-train 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['roofline']['frac'],4), 'C4', round(d['stress_c4']['value'],1))")"
done
