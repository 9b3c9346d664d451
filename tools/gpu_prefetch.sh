# trainer target prefetch: GPU tests, C2 bench block (device + e2e), multi-rank path
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-c4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_c2']; print('C3', round(d['value'],1), 'C2', round(t['value'],1), 'e2e', round(t['e2e']['value'],1))"
bash tools/gpu_multirank.sh 2>&1 | grep -E "rc="
