"""Bucket-size distribution of the depth sort on the C2 training cloud after
WARM iterations (development aid): how many buckets take the rank / mixed /
large paths of bucket_sort_depth."""
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
tr = Trainer(ds, GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0), device="cuda"),
             TrainConfig(iterations=20000, log_interval=10**9, eval_interval=10**9))
for _ in range(warm):
    tr.step()
torch.cuda.synchronize()
fr = tr.eng.frame
keys = fr.depth_key[: tr.cloud.n_points].cpu().numpy().view(np.uint64)
nt = fr.tiles_touched[: tr.cloud.n_points].cpu().numpy()
k = keys[nt > 0]
kmin, kmax = int(k.min()), int(k.max())
ln = (kmax - kmin).bit_length()
shift = max(ln - 16, 0)
b = np.minimum((k - np.uint64(kmin)) >> np.uint64(shift), 65534).astype(np.int64)
cnt = np.bincount(b, minlength=65535)
uniq = {}
order = np.argsort(b, kind="stable")
bs, ks = b[order], k[order]
starts = np.flatnonzero(np.r_[True, bs[1:] != bs[:-1]])
ends = np.r_[starts[1:], bs.size]
mixed = [(e - s, len(np.unique(ks[s:e]))) for s, e in zip(starts, ends) if e - s > 1 and len(np.unique(ks[s:e])) > 1]
sizes = np.array([m[0] for m in mixed]) if mixed else np.zeros(0)
d = k.view(np.float64)
print(f"depth range {d.min():.3f} .. {d.max():.3f}, quantiles {np.quantile(d, [0.001, 0.5, 0.999]).round(2)}, shift {shift}")
print(f"warm {warm}: N active {k.size}, buckets used {(cnt > 0).sum()}, max bucket {cnt.max()}, "
      f"mixed buckets {len(mixed)}: <=32 {int((sizes <= 32).sum())}, 33..256 {int(((sizes > 32) & (sizes <= 256)).sum())}, "
      f">256 {int((sizes > 256).sum())}; largest mixed {sizes.max() if sizes.size else 0}")
