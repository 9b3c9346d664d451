# checkpointed replay: GPU tests, then C2 training with each replay variant
set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for v in "" p2 p1; do echo "== variant [$v]"; XG_LIB_VARIANT=$v timeout 300 python tools/probe_train.py 300 2>&1 | tail -1; done
echo "== old path"; XG_BWD_CKPT=0 timeout 300 python tools/probe_train.py 300 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_train_ck.csv python tools/probe_train.py 10 > /dev/null 2>&1; echo "rc=$?"
