set -x
for k in k_preprocess k_bin_emit k_bin_count; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k\b|$k\(" -s 0 -c 1 -o gpurun_out/ncu_$k python tools/prof_c3.py 1 > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_os_pass -s 3 -c 1 -o gpurun_out/ncu_k_os_pass python tools/prof_c3.py 1 > gpurun_out/ncu_k_os_pass.log 2>&1; echo "os rc=$?"
