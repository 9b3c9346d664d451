"""Sweep throughput split for the batched renderer (development aid): full
sweep vs binning-only (12 streams, no compositing) vs compositing-only
(the 12-view launch over pre-binned frames), C3, ms per view."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native as nat  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.geometry import XgCamera  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, n_streams=4, batch=K)
out = torch.empty((360, 512, 512), device="cuda")
r.render(angles, out=out)
inten, inv = nat.intensities(cloud), nat.view_invariants(cloud)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * 360)


def full():
    r.render(angles, out=out, check=False)


def bin_only():
    main = torch.cuda.current_stream()
    for s in r.streams:
        s.wait_stream(main)
    for i, phi in enumerate(angles):
        st, fr = r.streams[i % K], r.frames[i % K]
        with torch.cuda.stream(st):
            fr.preprocess(cloud, r.camera(phi), inten, inv)
            fr.bin()
    for s in r.streams:
        main.wait_stream(s)


# frames binned once (first K views), composited 360/K times
fs = r.frames[:K]
for i in range(K):
    fs[i].preprocess(cloud, r.camera(angles[i]), inten, inv)
    fs[i].ensure_binned()
cams = (XgCamera * K)(*[f.cam for f in fs])
sps = (nat.XgSplats * K)(*[f.splats_struct() for f in fs])
imgs = (ctypes.c_void_p * K)(*[out[i].data_ptr() for i in range(K)])


def comp_only():
    for _ in range(360 // K):
        nat.lib().xg_composite_fwd_batch(cams, sps, imgs, K, r._batch_ws.data_ptr(), r._batch_ws.numel(),
                                         nat.stream())


for name, fn in (("full", full), ("bin", bin_only), ("comp", comp_only), ("full", full)):
    print(f"{name:5s} {timeit(fn):.4f} ms/view", flush=True)
