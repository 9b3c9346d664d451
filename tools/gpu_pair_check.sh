# streamed forward + replay pair: tests (guarded), A/B of iteration time, bench, C2 launch list
timeout 300 python -m pytest tests/test_gpu_train_pair.py tests/test_gpu_fused_loss.py -x -q > gpurun_out/pair_pytest.log 2>&1; rc=$?
echo "pair tests rc=$rc"; tail -15 gpurun_out/pair_pytest.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pair_pytest_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pair_pytest_all.log
for st in 0 1; do
  XG_TRAIN_STREAM=$st timeout 300 python tools/probe_train.py 1000 88 1000 2>&1 | tail -1
done
timeout 900 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/pair_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/pair_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_c2']; print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C2', round(t['value'],1), 'C2e2e', round(t['e2e']['value'],1), 'C4', round(d['stress_c4']['value'],1), 'C1', round(d['fwdbwd_c1']['value'],1), 'pair_ms', t['kernel_ms'], 'frac', t['roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/pair_launches_c2.csv python tools/probe_train.py 5 88 1000 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/pair_launches_c2.csv 5 | head -30
