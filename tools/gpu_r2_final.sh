# round-2 final evidence: round check (GPU tests, smoke, bench + CPU baselines, reference arm), then the
# launch list of one timed C3 step and of 200 timed C2 iterations (training pair), ncu --set full of the
# 12-view compositing launch, the pair's kernels inside the C2 timed window and the sweep emit
bash tools/gpu_r2_check.sh
XG_PROFILE_TIMED=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 20000 --csv \
    --log-file gpurun_out/r02_launches_timed_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-train --no-c4 --no-c1 > gpurun_out/r02_bench_ncu.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_timed_c3.csv 360 > gpurun_out/r02_launches_timed_c3_summary.txt; head -12 gpurun_out/r02_launches_timed_c3_summary.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 20000 --csv \
    --log-file gpurun_out/r02_launches_train_c2_pair.csv python tools/probe_train.py 200 88 1000 > /dev/null 2>&1; echo "train launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_train_c2_pair.csv 200 > gpurun_out/r02_launches_train_c2_pair_summary.txt; head -12 gpurun_out/r02_launches_train_c2_pair_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/r02_ncu_fwd_batch python tools/prof_batch.py 3 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_fwd_batch.ncu-rep > gpurun_out/r02_ncu_fwd_batch.txt 2>&1
bash tools/gpu_prof_pair.sh > /dev/null 2>&1; echo "pair rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_emit -c 1 \
    -o gpurun_out/r02_ncu_emit python tools/prof_c3.py 1 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_emit.ncu-rep > gpurun_out/r02_ncu_emit.txt 2>&1
head -14 gpurun_out/r02_ncu_fwd_batch.txt gpurun_out/r02_ncu_bwd_stream.txt gpurun_out/r02_ncu_fwd_pair.txt gpurun_out/r02_ncu_emit.txt
