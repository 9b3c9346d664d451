# ncu --set full of one onesweep pass, the bin emit and the preprocess at C3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_os_pass -s 3 -c 1 \
    -o gpurun_out/ncu_ospass python tools/prof_c3.py 1 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_emit -c 1 \
    -o gpurun_out/ncu_emit python tools/prof_c3.py 1 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_preprocess -c 1 \
    -o gpurun_out/ncu_pre python tools/prof_c3.py 1 > /dev/null 2>&1; echo "rc=$?"
