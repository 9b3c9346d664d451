# binning throughput (graph replay, 24 concurrent views) + C3/C4 bench + binning parity tests
timeout 100 python tools/probe_bin_graph.py 24 | tail -1
timeout 600 python -m pytest tests/test_gpu_reference_fullsize.py tests/test_gpu_parity.py -q -x -k "binning or bit_exact or sweep" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --no-train --no-c1 --no-c5 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], 'e2e', d['e2e']['value'], 'C4', d['stress_c4']['value'])"; done
