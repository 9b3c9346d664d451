# fused Adam + renorm check, C3 with the entry-balanced binning for every frame (XG_BIN_BALANCED=2) vs training frames only
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest.log
timeout 300 python tools/probe_train.py 2000 88 1000 2>&1 | tail -1
for b in 1 2; do
  XG_BIN_BALANCED=$b timeout 900 python bench.py --no-cpu-baseline --no-c5 --no-train > gpurun_out/r2b_bench_$b.log 2>&1; echo "bench $b rc=$?"
  tail -1 gpurun_out/r2b_bench_$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'rv', round(d['e2e']['render_view_loop']['value'],1), 'C4', round(d['stress_c4']['value'],1), 'C1', round(d['fwdbwd_c1']['value'],1))"
done
