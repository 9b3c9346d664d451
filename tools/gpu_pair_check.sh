# the overlapped training pair: its tests, the trainer tests, 4,000 C2 iterations, the bench (C2 / C3 / C4 / C1)
timeout 300 python -m pytest tests/test_gpu_train_pair.py tests/test_gpu_fused_loss.py tests/test_gpu_trainer.py -x -q > gpurun_out/pair_pytest.log 2>&1; rc=$?
echo "pair tests rc=$rc"; tail -3 gpurun_out/pair_pytest.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python tools/probe_train.py 4000 88 1000 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/pair_bench.log 2>&1; echo "bench rc=$?"
grep -v "^frame #" gpurun_out/pair_bench.log | grep -i "error\|Traceback" | head -5
tail -1 gpurun_out/pair_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_c2']; print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C2', round(t['value'],1), 'C2e2e', round(t['e2e']['value'],1), 'C4', round(d['stress_c4']['value'],1), 'C1', round(d['fwdbwd_c1']['value'],1), 'kms', t['kernel_ms'], 'frac', t['roofline']['frac'])"
