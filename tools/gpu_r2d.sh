# bucket sort with two memsets (was eight): GPU tests, C2 iteration times, C3 sweep
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2d_pytest.log
for i in 1 2 3; do timeout 300 python tools/probe_train.py 2000 88 1000 2>&1 | tail -1; done
timeout 900 python bench.py --no-cpu-baseline --no-c5 --no-c4 --no-c1 > gpurun_out/r2d_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2d_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_c2']; print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C2', round(t['value'],1), 'C2e2e', round(t['e2e']['value'],1))"
