"""Image-only compositing batches by path (row recurrence / direct EX2) over
C3 and C4 sweeps - needs the XG_BWD_STATS tuning build (development aid):
XG_LIB_VARIANT=bstats python tools/probe_fwd_stats.py."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import _native, acui, geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402

lib = _native.lib()
out = (ctypes.c_ulonglong * 8)()
for g, d in ((152, 512), (196, 1024)):
    cloud = GaussianCloud(**acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0), device="cuda")
    sc = geometry.ScannerConfig(1000.0, 1500.0, d, d, 192.0 / d)
    SweepRenderer(cloud, sc, batch=8).render(bench.sweep_angles(0, 1)[:16])
    torch.cuda.synchronize()
    lib.xg_debug_fwd_stats(out)
    b = list(out)
    print(f"G={g} D={d}: batches recurrence {b[0] / max(1, b[0] + b[1]):.3f} | survivors/batch rec "
          f"{b[2] / max(1, b[0]):.1f} direct {b[3] / max(1, b[1]):.1f} | batches with one half dead "
          f"{b[5] / max(1, b[4] + b[5]):.3f}, live lanes/batch {b[6] / max(1, b[4] + b[5]):.1f}")
