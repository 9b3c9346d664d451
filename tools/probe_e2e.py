"""C3 end-to-end overheads (development aid): the sweep with / without the
cloud upload and the image downloads."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
r = SweepRenderer(cloud, sc, n_streams=4, batch=12)
out = torch.empty((len(angles), 512, 512), device="cuda")
host = torch.empty((len(angles), 512, 512), pin_memory=True)
cloud_host = cloud.flat.detach().cpu().pin_memory()


def run(h2d, d2h, reps=5):
    for _ in range(2):
        r.render(angles, out=out, host_out=host if d2h else None, check=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        if h2d:
            cloud.flat.copy_(cloud_host, non_blocking=True)
        r.render(angles, out=out, host_out=host if d2h else None, check=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"h2d={h2d} d2h={d2h}: {ms:.2f} ms/step, {len(angles) / ms * 1e3:.0f} fps")


for h2d, d2h in ((False, False), (True, False), (False, True), (True, True)):
    run(h2d, d2h)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); host.copy_(out, non_blocking=True); t1.record(); torch.cuda.synchronize()
print(f"D2H {out.numel() * 4 / 1e6:.0f} MB alone: {t0.elapsed_time(t1):.2f} ms")
t0.record(); cloud.flat.copy_(cloud_host, non_blocking=True); t1.record(); torch.cuda.synchronize()
print(f"H2D {cloud_host.numel() * 4 / 1e6:.0f} MB alone: {t0.elapsed_time(t1):.2f} ms")
