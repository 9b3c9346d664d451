# C2 training-window diagnostics: workload statistics (tiles touched per splat, entries per binning warp,
# per-tile entries, replay walks, terminated pixels) + ncu of the binning kernels at iteration 1003
timeout 600 python tools/probe_c2_stats.py 88 1000 > gpurun_out/c2_stats.txt 2>&1; echo "stats rc=$?"; tail -14 gpurun_out/c2_stats.txt
for k in k_bin_emit k_bin_count k_scan; do
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -s 2 -c 1 \
    -o gpurun_out/c2_ncu_$k python tools/probe_train.py 8 88 1000 > /dev/null 2>&1; echo "$k rc=$?"
python tools/ncu_summary.py gpurun_out/c2_ncu_$k.ncu-rep > gpurun_out/c2_ncu_$k.txt 2>&1
head -24 gpurun_out/c2_ncu_$k.txt
done
