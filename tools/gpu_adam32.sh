# float32 Adam: trainer tests + C2 iteration
timeout 900 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_reference_ports.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do echo "C2 $(timeout 600 python tools/probe_train.py 400 2>&1 | tail -1)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_train.csv python tools/probe_train.py 10 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_train.csv 2>/dev/null | head -14
