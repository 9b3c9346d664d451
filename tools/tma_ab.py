"""TMA A/B (development aid): render 36 C3 views with the loaded library
(XG_LIB_VARIANT=tma selects the cp.async.bulk index-staging build), save the
stack (for a bit-for-bit comparison between builds) and time the batched sweep."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

out_path = sys.argv[1]
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, batch=12)
out = torch.empty((360, 512, 512), device="cuda")
r.render(angles, out=out)
np.save(out_path, out[::10].cpu().numpy())
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r.render(angles, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 360)
print(f"{out_path}: {best * 1e3:.1f} us/view (best of 5 sweeps)")
