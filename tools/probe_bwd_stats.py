"""Reverse-replay batches by path (exact / general / speculative) over C2
training iterations - needs the XG_BWD_STATS tuning build (development aid):
XG_LIB_VARIANT=bstats python tools/probe_bwd_stats.py [iters]."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native, acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, Trainer  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512, geometry.equal_interval_angles(100))
ds, _ = bench.phantom_dataset(88, sc)
tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(88), 16, 0), device="cuda"),
             TrainConfig(iterations=20000, log_interval=10**9, eval_interval=10**9))
lib = _native.lib()
out = (ctypes.c_ulonglong * 6)()
for chunk in range(4):
    for _ in range(iters // 4):
        tr.step()
    torch.cuda.synchronize()
    lib.xg_debug_bwd_stats(out)
    b = list(out)
    tot = max(1, sum(b[:3]))
    print(f"iters {(chunk + 1) * iters // 4}: batches exact {b[0] / tot:.3f} general {b[1] / tot:.3f} spec {b[2] / tot:.3f}"
          f" | survivors/batch exact {b[3] / max(1, b[0]):.1f} spec {b[5] / max(1, b[2]):.1f}")
