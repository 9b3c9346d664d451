"""Forward compositing variants on one C2 view (development aid): the
image-only split-half kernel vs the trainer's tracking forward, CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.engine import Frame  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 88
cloud = GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
fr = Frame(cloud.n_points, 512, 512, "cuda")
res = {"image_only": [], "train": [], "exact_track": []}
for phi in np.linspace(0.1, 3.0, 8):
    fr.preprocess(cloud, geometry.camera_pod(geometry.extrinsic_from_angle(sc, phi), geometry.intrinsic_from_config(sc),
                                             (512, 512)))
    fr.ensure_binned()
    for name, kw in (("image_only", dict(track=False)), ("train", dict(train=True)), ("exact_track", {})):
        fr.composite(**kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fr.composite(**kw)
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / 5)
print({k: f"{1e3 * np.mean(v):.1f} us" for k, v in res.items()})
