"""Termination statistics of the C2 training forward (development aid): after
WARM training iterations, the share of pixels whose transmittance falls below
the floor (n_contrib < tile length), the share of pairs past their pixel's
termination, and the image-only vs tracking forward times on that frame."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, Trainer  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
g = 88
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512, geometry.equal_interval_angles(100))
ds, _ = bench.phantom_dataset(g, sc)
tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0),
                               device="cuda"), TrainConfig(iterations=20000, log_interval=10**9,
                                                           eval_interval=10**9))
for _ in range(warm):
    tr.step()
torch.cuda.synchronize()
fr = tr.eng.frame


def timed(kw, n=10):
    fr.composite(**kw)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fr.composite(**kw)
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n


t_img = timed(dict(track=False))
t_train = timed(dict(train=True))
t_exact = timed({})
nc = fr.n_contrib.cpu().numpy().astype(np.int64)
tf = fr.t_final.cpu().numpy()
rng = fr.tile_ranges.cpu().numpy()
h, w = nc.shape
ty, tx = np.meshgrid(np.arange(h) // 16, np.arange(w) // 16, indexing="ij")
tl = (rng[:, 1] - rng[:, 0])[ty * ((w + 15) // 16) + tx]
term = tf < 1e-4
print(f"N={tr.cloud.n_points} entries={int(rng[-1, 1])} mean tile len {tl.mean():.0f}")
print(f"terminated pixels {term.mean() * 100:.2f} %; pairs traversed {nc.sum():.3e} of {tl.sum():.3e} "
      f"({100 * nc.sum() / tl.sum():.1f} %); pairs past termination {100 * (tl - nc)[term].sum() / tl.sum():.2f} %")
print(f"forward: image-only {t_img:.1f} us, train {t_train:.1f} us, exact tracking {t_exact:.1f} us")
chunks = np.ceil((rng[:, 1] - rng[:, 0]) / 256).astype(int)
print(f"256-entry chunks per tile: mean {chunks.mean():.1f}, max {chunks.max()}, total {chunks.sum()}")
