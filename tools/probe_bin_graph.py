"""GPU-side throughput of the sweep's binning (development aid): the
preprocess + xg_bin_sort of 12 views on 12 streams captured once in a CUDA
graph (no host launch cost), replayed; compare with the batched sweep's
per-batch gap (tools/probe_timeline.py).  usage: [XG_BIN_STOP=k] probe_bin_graph.py [K] [pre]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native as nat  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.engine import Frame  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
PRE_ONLY = len(sys.argv) > 2 and sys.argv[2] == "pre"  # preprocess only (else XG_BIN_STOP=k cuts xg_bin_sort)
cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, n_streams=4, batch=12)
r.prepare(angles)  # (no compositing: XG_BIN_STOP leaves the lists incomplete)
torch.cuda.synchronize()
inten, inv = nat.intensities(cloud), nat.view_invariants(cloud)
streams = [torch.cuda.Stream() for _ in range(K)]
frames = [Frame(cloud.n_points, 512, 512, "cuda", entry_capacity=r.capacity) for _ in range(K)]


def body():
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for i in range(K):
        with torch.cuda.stream(streams[i]):
            frames[i].preprocess(cloud, r.camera(angles[30 + i]), inten, inv)
            if not PRE_ONLY:
                frames[i].bin()
    for s in streams:
        main.wait_stream(s)


body()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.stream(cap):
    with torch.cuda.graph(g, stream=cap):
        body()
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"K={K}: graph replay {a.elapsed_time(b) / 20:.3f} ms per {K} views = us/view {a.elapsed_time(b) / 20 / K * 1e3:.1f}")
