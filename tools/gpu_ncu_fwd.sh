set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_fwd -s 2 -c 1 \
    -o gpurun_out/ncu_fwd python tools/probe.py 152 512 3 > gpurun_out/ncu_fwd.log 2>&1; echo "rc=$?"
