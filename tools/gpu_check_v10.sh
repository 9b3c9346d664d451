# quick check: bench line (roofline_hbm), multi-rank path on one GPU
timeout 900 python bench.py --no-cpu-baseline --no-train > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d.get('roofline_hbm'))"
bash tools/gpu_multirank.sh 2>&1 | grep -v "^+"
