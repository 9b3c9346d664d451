# view-invariant cache: GPU tests, C3 / C4 sweep
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-train > gpurun_out/bench_inv.log 2>&1; tail -1 gpurun_out/bench_inv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],4), 'C4', round(d['stress_c4']['value'],1), d['stress_c4']['stages_ms_isolated'])"
