"""Marginal cost of each binning stage inside a concurrent 12-stream C3
binning sweep (development aid; needs the XG_BIN_STOP hook of xg_bin_sort).
usage: XG_BIN_STOP=k python tools/probe_bin_stages.py [mode]
mode: pre (preprocess only) | bin (preprocess + xg_bin_sort up to XG_BIN_STOP)"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native as nat  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "bin"
K = 12
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, n_streams=4, batch=K)
r.prepare(angles)
inten, inv = nat.intensities(cloud), nat.view_invariants(cloud)


def run():
    main = torch.cuda.current_stream()
    for s in r.streams:
        s.wait_stream(main)
    for i, phi in enumerate(angles):
        st, fr = r.streams[i % K], r.frames[i % K]
        with torch.cuda.stream(st):
            fr.preprocess(cloud, r.camera(phi), inten, inv)
            if mode == "bin":
                fr.bin()
    for s in r.streams:
        main.wait_stream(s)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    run()
e1.record()
torch.cuda.synchronize()
print(f"{mode} stop={__import__('os').environ.get('XG_BIN_STOP', '0')}: {e0.elapsed_time(e1) / (3 * 360) * 1e3:.1f} us/view")
