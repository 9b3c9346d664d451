# ncu captures of the current kernels (round-1 profiles): launch list of one
# C3 view + training pass, and --set full of the top kernels.
set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv python tools/prof_c3.py 3 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd -s 2 -c 1 \
    -o gpurun_out/ncu_fwd python tools/prof_c3.py 3 > gpurun_out/ncu_fwd.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_bwd -s 2 -c 1 \
    -o gpurun_out/ncu_bwd python tools/prof_c3.py 3 > gpurun_out/ncu_bwd.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_os_pass -s 8 -c 1 \
    -o gpurun_out/ncu_sort python tools/prof_c3.py 1 > gpurun_out/ncu_sort.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_emit -s 1 -c 1 \
    -o gpurun_out/ncu_emit python tools/prof_c3.py 1 > gpurun_out/ncu_emit.log 2>&1; echo "rc=$?"
