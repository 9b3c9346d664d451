timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_emit -c 1 \
    -o gpurun_out/ncu_emit_c4 python tools/prof_c3.py 1 196 1024 > /dev/null 2>&1; echo "rc=$?"
