for v in ${VARIANTS:-base}; do echo -n "$v: "; XG_LIB_VARIANT=$v timeout 600 python -c "
import sys, types, json, torch
sys.path.insert(0, '.')
import bench
args = types.SimpleNamespace(streams=4, warmup=3, steps=3)
def timed(fn, k):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
r = bench.c4_block(args, timed, 1, 0)
print(round(r['value'],1), json.dumps(r['stages_ms_isolated']))
"; done
