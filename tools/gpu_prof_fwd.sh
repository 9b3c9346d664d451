# ncu --set full of the 12-view image-only compositing launch (C3)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd_batch -s 2 -c 1 \
    -o gpurun_out/r02_ncu_fwd_batch_v2 python tools/prof_batch.py 3 > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/r02_ncu_fwd_batch_v2.ncu-rep > gpurun_out/r02_ncu_fwd_batch_v2.txt 2>&1; head -24 gpurun_out/r02_ncu_fwd_batch_v2.txt
