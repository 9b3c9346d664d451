"""Per-iteration wall times around density-control events (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, Trainer  # noqa: E402

g = 88
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512, geometry.equal_interval_angles(100))
ds, _ = bench.phantom_dataset(g, sc)
for rep in range(2):
    tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0),
                                   device="cuda"), TrainConfig(iterations=20000, log_interval=10**9,
                                                               eval_interval=10**9))
    for _ in range(500):
        tr.step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        tr.step()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e3
    ev = [i for i in range(300) if (501 + i) % 100 == 0]
    print(f"trainer {rep}: median {np.median(ts):.3f} ms, densify iters {[round(ts[i], 2) for i in ev]} ms, "
          f"total {ts.sum():.1f} ms, N={tr.cloud.n_points}")
