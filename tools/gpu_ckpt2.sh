# chunk-size variants of the checkpointed replay (C2 training) + the new test
set -x
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "chunked or backward" 2>&1 | tail -3
for v in "" c128 c512 c1024; do echo "== variant [$v]"; XG_LIB_VARIANT=$v timeout 300 python tools/probe_train.py 300 2>&1 | tail -1; done
