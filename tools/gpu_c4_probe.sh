# C4 launch list (one view: preprocess, bin, tracked + image-only composite, backward)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python tools/prof_c3.py 1 196 1024 > /dev/null 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4.csv 2>/dev/null | head -24
