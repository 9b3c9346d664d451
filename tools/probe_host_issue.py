"""Host issue time vs device time of a C3 sweep (development aid): is the
batched sweep bound by the GPU or by the host's launch rate?
usage: python tools/probe_host_issue.py [mode]; mode: full | bin (XG_BIN_STOP-free,
binning + preprocess only, no compositing) | pre"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "full"
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, n_streams=4, batch=12)
r.render(angles)
torch.cuda.synchronize()
from paper_2403_04116_b200 import _native as nat  # noqa: E402

inten, inv = nat.intensities(cloud), nat.view_invariants(cloud)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "full":
        r.render(angles, check=False)
    else:
        main = torch.cuda.current_stream()
        for s in r.streams:
            s.wait_stream(main)
        for i, phi in enumerate(angles):
            st, fr = r.streams[i % len(r.streams)], r.frames[i % 12]
            with torch.cuda.stream(st):
                fr.preprocess(cloud, r.camera(phi), inten, inv)
                if mode == "bin":
                    fr.bin()
        for s in r.streams:
            main.wait_stream(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    n = len(angles)
    print(f"{mode}: host issue {1e3 * (t1 - t0) / n:.3f} ms/view, total {1e3 * (t2 - t0) / n:.3f} ms/view")
