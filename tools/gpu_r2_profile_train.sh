# ncu --set full of the training kernels INSIDE the bench's timed window
# (iteration 1001+: --profile-from-start off, probe_train.py starts the
# profiler after 1000 warm-up iterations)
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_bwd_ck -s 2 -c 1 \
    -o gpurun_out/r02_ncu_bwd_train python tools/probe_train.py 4 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_bwd_train.ncu-rep > gpurun_out/r02_ncu_bwd_train.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_fwd_np -s 2 -c 1 \
    -o gpurun_out/r02_ncu_fwdtrain python tools/probe_train.py 4 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_fwdtrain.ncu-rep > gpurun_out/r02_ncu_fwdtrain.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_preprocess_bwd -s 2 -c 1 \
    -o gpurun_out/r02_ncu_prebwd python tools/probe_train.py 4 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_prebwd.ncu-rep > gpurun_out/r02_ncu_prebwd.txt 2>&1
head -24 gpurun_out/r02_ncu_bwd_train.txt gpurun_out/r02_ncu_fwdtrain.txt gpurun_out/r02_ncu_prebwd.txt
