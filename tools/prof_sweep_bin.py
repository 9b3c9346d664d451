"""C3 sweep binning launches for ncu (development aid): a 12-view batch of the
bench's SweepRenderer path (view-invariant cache, bucket depth sort,
multisplit binning), rendered twice - profile the second with --launch-skip."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
r = SweepRenderer(cloud, sc, n_streams=1, batch=12)
angles = bench.sweep_angles(0, 1)[:12]
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r.render(angles)
torch.cuda.synchronize()
