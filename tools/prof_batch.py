"""Multi-view compositing launches for ncu (development aid): C3, 12 views
(the bench's launch size) binned, then `reps` xg_composite_fwd_batch launches."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)[:12]
r = SweepRenderer(cloud, sc, batch=12)
out = torch.empty((12, 512, 512), device="cuda")
for _ in range(reps):
    r.render(angles, out=out)
torch.cuda.synchronize()
