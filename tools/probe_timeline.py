"""Device timeline of the batched C3 sweep (development aid): CUDA events at
each view's binning start / end (its stream) and each compositing launch
(composite stream), relative to one start event - when does batch j's
binning run against batch j-1's compositing?"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native as nat  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.geometry import XgCamera  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
K = 12
r = SweepRenderer(cloud, sc, n_streams=4, batch=K)
out = r.render(angles)
torch.cuda.synchronize()
inten, inv = nat.intensities(cloud), nat.view_invariants(cloud)
lib = nat.lib()
D2H = len(sys.argv) > 1 and sys.argv[1] == "d2h"  # each batch's images to pinned host memory (copy stream)
host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
cps = torch.cuda.Stream()


def E():
    return torch.cuda.Event(enable_timing=True)


for rep in range(2):
    main = torch.cuda.current_stream()
    t0 = E()
    t0.record(main)
    cs = r.comp_stream
    for s in r.streams + [cs]:
        s.wait_stream(main)
    done = [None, None]
    rec = []
    for j, lo in enumerate(range(0, len(angles), K)):
        hi = min(lo + K, len(angles))
        fs = r.frames[(j % 2) * K:(j % 2) * K + K]
        bins = []
        for i in range(lo, hi):
            st, fr = r.streams[i - lo], fs[i - lo]
            with torch.cuda.stream(st):
                if done[j % 2] is not None:
                    st.wait_event(done[j % 2])
                a, b = E(), E()
                a.record(st)
                fr.preprocess(cloud, r.camera(angles[i]), inten, inv)
                fr.bin()
                b.record(st)
                bins.append((a, b))
            cs.wait_stream(st)
        nv = hi - lo
        cams = (XgCamera * nv)(*[fs[i].cam for i in range(nv)])
        sps = (nat.XgSplats * nv)(*[fs[i].splats_struct() for i in range(nv)])
        imgs = (ctypes.c_void_p * nv)(*[out[lo + i].data_ptr() for i in range(nv)])
        with torch.cuda.stream(cs):
            a, b = E(), E()
            a.record(cs)
            nat.check(lib.xg_composite_fwd_batch(cams, sps, imgs, nv, r._batch_ws.data_ptr(), r._batch_ws.numel(),
                                                 nat.stream()), "batch")
            b.record(cs)
            ev = torch.cuda.Event()
            ev.record(cs)
            done[j % 2] = ev
        if D2H:
            cps.wait_event(ev)
            with torch.cuda.stream(cps):
                host[lo:hi].copy_(out[lo:hi], non_blocking=True)
        rec.append((bins, (a, b)))
    for s in r.streams + [cs, cps]:
        main.wait_stream(s)
    te = E()
    te.record(main)
    torch.cuda.synchronize()
    if rep == 0:
        continue
    for j, (bins, (a, b)) in enumerate(rec):
        bs = [t0.elapsed_time(x) for x, _ in bins]
        be = [t0.elapsed_time(y) for _, y in bins]
        print(f"batch {j:2d}: bin {min(bs):7.3f} .. {max(be):7.3f} (first view done {min(be):7.3f}) | "
              f"comp {t0.elapsed_time(a):7.3f} .. {t0.elapsed_time(b):7.3f} ({a.elapsed_time(b):.3f})")
    print(f"total {t0.elapsed_time(rec[-1][1][1]):.3f} ms for {len(angles)} views (end incl. copies {t0.elapsed_time(te):.3f})")
    print("mean composite ms", sum(a.elapsed_time(b) for _, (a, b) in rec) / len(rec))
    gaps = [rec[j][1][1].elapsed_time(rec[j + 1][1][0]) for j in range(len(rec) - 1)]
    print("mean gap between compositing launches ms", sum(gaps) / len(gaps))
