# ncu --set full of the training pair's kernels inside the C2 timed window (iteration 1003) + launch list
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_bwd_stream -s 2 -c 1 \
    -o gpurun_out/r02_ncu_bwd_stream python tools/probe_train.py 8 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_bwd_stream.ncu-rep > gpurun_out/r02_ncu_bwd_stream.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_fwd_np -s 2 -c 1 \
    -o gpurun_out/r02_ncu_fwd_pair python tools/probe_train.py 8 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_fwd_pair.ncu-rep > gpurun_out/r02_ncu_fwd_pair.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_train_c2_pair.csv python tools/probe_train.py 5 88 1000 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_train_c2_pair.csv 5 > gpurun_out/r02_launches_train_c2_pair_summary.txt
head -20 gpurun_out/r02_ncu_bwd_stream.txt gpurun_out/r02_ncu_fwd_pair.txt; cat gpurun_out/r02_launches_train_c2_pair_summary.txt | head -30
