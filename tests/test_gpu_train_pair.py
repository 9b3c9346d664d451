"""xg_composite_train_pair (the trainer's overlapped forward + reverse
replay, streamed through a device ring) against the sequential pair it
replaces - xg_composite_fwd_train then xg_composite_bwd(dl_dimage = NULL) -
on a multi-chunk training scene: image, t_final, n_contrib, checkpoints and
the L1 sum bit-identical (the forward kernel is the same), the gradient
accumulator equal up to float-atomic summation order (1e-5 normwise).  Also
an entry-buffer overflow (the forward skips, the replay must end, not wait)
and the Trainer end to end on the pair."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise_ok

pytestmark = pytest.mark.gpu


def _setup(spec=48, det=256, phi=0.9, seed=0):
    import torch

    from paper_2403_04116_b200 import acui, geometry
    from paper_2403_04116_b200.gaussians import GaussianCloud
    from paper_2403_04116_b200.geometry import camera_pod
    from paper_2403_04116_b200.trainer import _IterationEngine

    arrs = acui.init_alternative_arrays("cuboid", acui.benchmark_spec(spec), 16, seed)
    cloud = GaussianCloud(**arrs, device="cuda")
    sc = geometry.ScannerConfig(1000.0, 1500.0, det, det, 192.0 / det)
    cam = camera_pod(geometry.extrinsic_from_angle(sc, phi), geometry.intrinsic_from_config(sc), (det, det))
    eng = _IterationEngine(cloud, det, det)
    tgt = (torch.rand((det, det), generator=torch.Generator().manual_seed(seed)) * 0.5).cuda().contiguous()
    return cloud, cam, eng, tgt


def _run(cloud, cam, eng, tgt, pair: bool):
    import torch

    fr = eng.frame
    h, w = fr.h, fr.w
    fr.preprocess(cloud, cam)
    fr.ensure_binned()
    if pair:
        fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
    else:
        fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        import ctypes

        from paper_2403_04116_b200 import _native as nat

        sp = fr.splats_struct()
        nat.check(nat.lib().xg_composite_bwd(ctypes.byref(fr.cam), ctypes.byref(sp), fr.t_final.data_ptr(),
                                             fr.n_contrib.data_ptr(), None, fr.image.data_ptr(), tgt.data_ptr(),
                                             ctypes.c_float(1.0 / (h * w)), eng.acc.data_ptr(), nat.stream()),
                  "xg_composite_bwd")
    torch.cuda.synchronize()
    return {"image": fr.image.clone(), "t_final": fr.t_final.clone(), "n_contrib": fr.n_contrib.clone(),
            "l1": float(eng.l1.item()), "acc": eng.acc[: cloud.n_points].clone(),
            "entries": int(fr.read_counters()[1])}


def test_train_pair_equals_sequential():
    import torch

    cloud, cam, eng, tgt = _setup()
    seq = _run(cloud, cam, eng, tgt, pair=False)
    par = _run(cloud, cam, eng, tgt, pair=True)
    assert seq["entries"] > 256 * 200, seq["entries"]  # tiles with several replay chunks
    for k in ("image", "t_final", "n_contrib"):
        assert torch.equal(seq[k], par[k]), k
    assert seq["l1"] == par["l1"] or abs(seq["l1"] - par["l1"]) <= 1e-12 * abs(seq["l1"])
    a, b = seq["acc"].cpu().numpy().astype(np.float64), par["acc"].cpu().numpy().astype(np.float64)
    for c in range(7):
        ok, rel = normwise_ok(b[:, c], a[:, c], 1e-3 * np.abs(a[:, c]).max() + 1e-30, tol=1e-5)
        assert ok, (c, rel)
    # repeated pairs on the same frame (epoch tags keep the ring's stale slots out)
    for _ in range(3):
        again = _run(cloud, cam, eng, tgt, pair=True)
        assert torch.equal(again["image"], par["image"])
        ok, rel = normwise_ok(again["acc"].cpu().numpy().astype(np.float64)[:, 0], a[:, 0],
                              1e-3 * np.abs(a[:, 0]).max() + 1e-30, tol=1e-5)
        assert ok, rel


def test_train_pair_entry_overflow_ends():
    """A too-small entry buffer: the forward skips every tile, publishes no
    chunks, and the replay grid must exit (finish_bin then re-bins and the
    second pair runs for real)."""
    import torch

    cloud, cam, eng, tgt = _setup(spec=32, det=128)
    ref = _run(cloud, cam, eng, tgt, pair=True)
    assert ref["entries"] > 4096
    eng.resize(cloud, capacity=1024)  # (a fresh frame whose entry buffer is too small)
    fr = eng.frame
    h, w = fr.h, fr.w
    fr.preprocess(cloud, cam)
    fr.bin_async()
    fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
    torch.cuda.synchronize()  # (hangs here if the replay waited for chunks that never come)
    assert fr.finish_bin()
    fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
    torch.cuda.synchronize()
    assert torch.equal(fr.image, ref["image"])
    a, b = ref["acc"].cpu().numpy().astype(np.float64), eng.acc[: cloud.n_points].cpu().numpy().astype(np.float64)
    ok, rel = normwise_ok(b[:, 0], a[:, 0], 1e-3 * np.abs(a[:, 0]).max() + 1e-30, tol=1e-5)
    assert ok, rel
