set -x
timeout 600 python tools/probe_train.py 200 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_train.csv python tools/probe_train.py 10 > /dev/null 2>&1; echo "rc=$?"
