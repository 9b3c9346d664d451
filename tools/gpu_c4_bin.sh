# C4 binning: fused multisplit (T = 4096) vs duplicate + radix sort by tile
for v in base ms1k base ms1k; do
  if [ $v = base ]; then unset XG_LIB_VARIANT; else export XG_LIB_VARIANT=$v; fi
  echo "$v $(timeout 300 python tools/probe.py 196 1024 8 2>&1 | grep 'per view')"
done
export XG_LIB_VARIANT=ms1k
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4_ms1k.csv python tools/prof_c3.py 1 196 1024 > /dev/null 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4_ms1k.csv 2>/dev/null | head -20
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -2
