# ncu --set full of the C2 reverse replay and tracking forward inside the
# timed window (iterations 1001+: --profile-from-start off, probe_train.py
# opens the profiler range after its warm-up)
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_bwd_ck -s 2 -c 1 \
    -o gpurun_out/r02_ncu_bwd_timed python tools/probe_train.py 8 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_bwd_timed.ncu-rep > gpurun_out/r02_ncu_bwd_timed.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_composite_fwd_np -s 2 -c 1 \
    -o gpurun_out/r02_ncu_fwdtrain_timed python tools/probe_train.py 8 88 1000 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_fwdtrain_timed.ncu-rep > gpurun_out/r02_ncu_fwdtrain_timed.txt 2>&1
head -24 gpurun_out/r02_ncu_bwd_timed.txt gpurun_out/r02_ncu_fwdtrain_timed.txt
