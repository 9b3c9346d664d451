"""Sweep throughput split (development aid): full sweep vs binning-only vs
composite-only, 4 streams, C3."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
r = SweepRenderer(cloud, sc, n_streams=ns)
out = torch.empty((360, 512, 512), device="cuda")
r.render(angles, out=out)


def run(mode):
    main = torch.cuda.current_stream()
    for s in r.streams:
        s.wait_stream(main)
    for i, phi in enumerate(angles):
        k = i % len(r.streams)
        with torch.cuda.stream(r.streams[k]):
            fr = r.frames[k]
            if mode in ("full", "bin"):
                fr.preprocess(cloud, r.camera(phi))
                fr.bin()
            if mode in ("full", "comp"):
                fr.composite(image_out=out[i], track=False)
    for s in r.streams:
        main.wait_stream(s)


for mode in ("full", "bin", "comp", "full"):
    run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run(mode)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode:5s} {e0.elapsed_time(e1) / (3 * 360):.4f} ms/view")
