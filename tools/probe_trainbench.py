"""Run bench.train_block twice (development aid: device vs e2e ordering)."""
import sys
import types

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

args = types.SimpleNamespace(warmup=3, steps=5, train_iters_per_step=100)


def timed(fn, k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(2):
    r = bench.train_block(args, timed, bench.ClockSampler, 0, 1)
    print(rep, "device", round(r["value"], 1), "e2e", round(r["e2e"]["value"], 1))
