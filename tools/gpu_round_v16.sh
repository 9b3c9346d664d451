# round check: GPU tests, smoke, bench (+ reference arm), launch list of the timed sweep, ncu of the top kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-800
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
XG_PROFILE_TIMED=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 20000 --csv \
    --log-file gpurun_out/launches_timed.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-train --no-c4 > gpurun_out/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_timed.csv 2>/dev/null | head -16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/ncu_fwd_batch python tools/prof_batch.py 3 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd_ck -s 30 -c 1 \
    -o gpurun_out/ncu_bwd_train python tools/probe_train.py 40 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_np -s 30 -c 1 \
    -o gpurun_out/ncu_fwdtrain python tools/probe_train.py 40 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_emit -c 1 \
    -o gpurun_out/ncu_emit python tools/prof_c3.py 1 > /dev/null 2>&1; echo "rc=$?"
