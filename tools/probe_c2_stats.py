"""C2 training window statistics (development aid): per-Gaussian tiles
touched, per-tile entries and per-quarter replay cost after WARM iterations,
plus the binning warps' entry imbalance (one 32-Gaussian round per warp)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.trainer import TrainConfig, Trainer  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 88
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512, geometry.equal_interval_angles(100))
ds, _ = bench.phantom_dataset(g, sc)
tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0),
                               device="cuda"), TrainConfig(iterations=20000, log_interval=10**9,
                                                           eval_interval=10**9))
for _ in range(warm + 1):  # (+1: iteration warm is a density-control event; the next one rebinds the frame)
    tr.step()
torch.cuda.synchronize()
fr = tr.eng.frame


def pct(a, name):
    a = np.sort(np.asarray(a, np.float64))
    q = [50, 90, 99, 99.9, 100]
    print(f"{name}: n={a.size} mean={a.mean():.1f} " + " ".join(f"p{x}={np.percentile(a, x):.0f}" for x in q)
          + f" sum={a.sum():.0f}")


tt = fr.tiles_touched.cpu().numpy()[: fr.n]
pct(tt, "tiles touched / Gaussian")
order = fr.order.cpu().numpy()[: fr.n]
tt_sorted = tt[order]
w = tt_sorted[: (tt_sorted.size // 32) * 32].reshape(-1, 32).sum(1)
pct(w, "entries / binning warp (32 depth-sorted Gaussians)")
cta = tt_sorted[: (tt_sorted.size // 256) * 256].reshape(-1, 256).sum(1)
pct(cta, "entries / binning CTA (256 Gaussians)")
r = fr.tile_ranges.cpu().numpy()
pct(r[:, 1] - r[:, 0], "entries / tile")
uc = fr.unit_cost.cpu().numpy()
pct(uc, "replay walk / quarter (unit_cost)")
print("max tile entries / mean:", (r[:, 1] - r[:, 0]).max() / (r[:, 1] - r[:, 0]).mean())
tf = fr.t_final.cpu().numpy()
nc = fr.n_contrib.cpu().numpy()
print(f"terminated pixels (t_final < 1e-4): {np.mean(tf < 1e-4):.3f}")
# per-tile: the terminated share and walk length vs list length
ntx = (fr.w + 15) // 16
ln = (r[:, 1] - r[:, 0]).reshape(-1, ntx)
ncm = nc.reshape(fr.h // 16, 16, ntx, 16).max(axis=(1, 3))
heavy = ln >= np.percentile(ln, 90)
print(f"heaviest 10 % tiles: mean list {ln[heavy].mean():.0f}, mean max walk {ncm[heavy].mean():.0f}, "
      f"terminated px {np.mean((tf.reshape(fr.h // 16, 16, ntx, 16) < 1e-4).mean(axis=(1, 3))[heavy]):.3f}")
