# A/B of the entry-balanced binning (XG_BIN_BALANCED=1, default) vs the Gaussian-chunked count / emit
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/bal_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/bal_pytest.log
for b in 0 1; do
  XG_BIN_BALANCED=$b timeout 300 python tools/probe_train.py 1000 88 1000 2>&1 | tail -1
done
for b in 0 1; do
  XG_BIN_BALANCED=$b timeout 900 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/bal_bench_$b.log 2>&1; echo "bench $b rc=$?"
  tail -1 gpurun_out/bal_bench_$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'C2', round(d['train_c2']['value'],1), 'C4', round(d['stress_c4']['value'],1), 'C1', round(d['fwdbwd_c1']['value'],1))"
done
nsys_dummy=0
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/bal_launches_c2.csv python tools/probe_train.py 5 88 1000 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/bal_launches_c2.csv 5 | head -30
