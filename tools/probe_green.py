"""SM-partitioned sweep (development aid): binning streams on a green context
of B SMs, the batched compositing stream on the remaining SMs, vs the
default shared-SM sweep.  C3, ms per view.  usage: probe_green.py B [B ...]"""
import sys

import numpy as np
import torch
from cuda.bindings import driver as drv

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_04116_b200 import geometry  # noqa: E402
from paper_2403_04116_b200.gaussians import GaussianCloud  # noqa: E402
from paper_2403_04116_b200.inference import SweepRenderer  # noqa: E402


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    assert err == drv.CUresult.CUDA_SUCCESS, err
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


torch.zeros(1, device="cuda")
dev = ok(drv.cuDeviceGet(0))
sm_res = ok(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("SMs:", sm_res.sm.smCount, flush=True)


def green_streams(bin_sms: int, n_bin_streams: int):
    groups, nb, rem = ok(drv.cuDevSmResourceSplitByCount(1, sm_res, 0, bin_sms))
    g_bin = groups[0] if isinstance(groups, (list, tuple)) else groups
    print(f"  split: bin {g_bin.sm.smCount} SMs, rest {rem.sm.smCount} SMs", flush=True)
    out = []
    for res, n in ((g_bin, n_bin_streams), (rem, 1)):
        desc = ok(drv.cuDevResourceGenerateDesc([res], 1))
        gctx = ok(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        ss = []
        for _ in range(n):
            s = ok(drv.cuGreenCtxStreamCreate(gctx, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
            ss.append(torch.cuda.ExternalStream(int(s)))
        out.append(ss)
    return out[0], out[1][0]


cloud = GaussianCloud(**bench.c3_arrays(), device="cuda")
sc = geometry.ScannerConfig(1000.0, 1500.0, 512, 512, 192.0 / 512)
angles = bench.sweep_angles(0, 1)
K = 12
out = torch.empty((360, 512, 512), device="cuda")


def timeit(r, reps=3):
    r.render(angles, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r.render(angles, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * 360)


base = SweepRenderer(cloud, sc, batch=K)
ref_img = None
print(f"shared   {timeit(base):.4f} ms/view", flush=True)
ref_img = out.clone()
for b in [int(x) for x in sys.argv[1:]]:
    r = SweepRenderer(cloud, sc, batch=K)
    r.streams, r.comp_stream = green_streams(b, K)
    t = timeit(r)
    same = torch.equal(out, ref_img)
    print(f"green {b:3d} {t:.4f} ms/view  (images identical: {same})", flush=True)
