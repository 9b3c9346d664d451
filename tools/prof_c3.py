"""Minimal C3 launches for ncu (development aid): one view binned, then
`reps` image-only composites (the bench's kernel) and `reps` tracked
composites + backward passes (the training path)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_04116_b200 import acui, geometry  # noqa: E402
from paper_2403_04116_b200.engine import Frame  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402


def main(reps=3, g=152, d=512):
    cloud = GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0), device="cuda")
    sc = geometry.ScannerConfig(1000.0, 1500.0, d, d, 192.0 / d)
    cam = geometry.camera_pod(geometry.extrinsic_from_angle(sc, 0.7), geometry.intrinsic_from_config(sc), (d, d))
    fr = Frame(cloud.n_points, d, d, "cuda", entry_capacity=30 * cloud.n_points)
    fr.preprocess(cloud, cam)
    fr.ensure_binned()
    for _ in range(reps):
        fr.composite(track=False)
    acc = torch.zeros((cloud.n_points, 8), device="cuda")
    gflat = torch.empty_like(cloud.flat)
    sn = torch.empty(cloud.n_points, device="cuda")
    vis = torch.empty(cloud.n_points, dtype=torch.uint8, device="cuda")
    dl = torch.as_tensor(np.random.default_rng(0).normal(size=(d, d)) / (d * d), dtype=torch.float32, device="cuda")
    for _ in range(reps):
        fr.composite(track=True)
        fr.backward(cloud, acc, gflat, sn, vis, dl_dimage=dl)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
