"""Run a few C2 training iterations (development aid, for ncu launch lists)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, Trainer  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = int(sys.argv[2]) if len(sys.argv) > 2 else 88
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 5  # 1000: the bench's timed window (iterations 1001..)
reproducible = len(sys.argv) > 4 and sys.argv[4] == "reproducible"
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512, geometry.equal_interval_angles(100))
ds, _ = bench.phantom_dataset(g, sc)
tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0),
                               device="cuda"), TrainConfig(iterations=20000, log_interval=10**9,
                                                           eval_interval=10**9), reproducible=reproducible)
for _ in range(warm):
    tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures only these iterations
t0 = time.perf_counter()
for _ in range(iters):
    tr.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{iters} iterations: {1e3 * (time.perf_counter() - t0) / iters:.3f} ms/iter, N={tr.cloud.n_points}, "
      f"entries={getattr(tr.eng.frame, 'last_counters', [0, -1])[1]}")
