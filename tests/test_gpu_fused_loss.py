"""The trainer's fused training objective against the REAL reference
(tests/golden/l1.npz, make_golden_l1.py): the L1 sum accumulated inside the
tracking forward (``xg_composite_fwd_train``'s ``l1_sum``) and the
sign(I - target) / HW upstream formed inside the reverse replay
(``xg_composite_bwd``'s ``target`` + ``l1_scale``) - the exact calls
``Trainer.step`` makes at gamma = 0 - and, at gamma = 0.2, the
``xg_ssim``-written dL/dI feeding the same backward; versus the reference's
``loss(rendered, target, gamma)`` (trainer.py:109-123) followed by
``render_backward`` (backward.py:21-124).  Loss within 1e-6 relative,
RenderGradients normwise within 1e-4."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from conftest import normwise_ok

pytestmark = pytest.mark.gpu

L1 = Path(__file__).resolve().parent / "golden" / "l1.npz"
FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")


@pytest.fixture(scope="module")
def l1g():
    d = np.load(L1)
    return {k: d[k] for k in d.files}


def _scene(golden, name):
    import torch

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.geometry import camera_pod
    from paper_2403_04116_b200.trainer import DensifyStats, _IterationEngine

    p = name + "/"
    cloud = xg.GaussianCloud(**{f: golden[p + f] for f in FIELDS}, basis_weights=golden[p + "basis_weights"],
                             device="cuda")
    l_so, l_sd, w, h, pitch, phi = golden[p + "camera"]
    w, h = int(w), int(h)
    sc = xg.ScannerConfig(l_so, l_sd, w, h, pitch)
    cam = camera_pod(xg.extrinsic_from_angle(sc, phi), xg.intrinsic_from_config(sc), (h, w))
    eng = _IterationEngine(cloud, h, w)
    stats = DensifyStats.zeros(cloud.n_points, cloud.device)
    torch.cuda.synchronize()
    return cloud, cam, eng, stats, h, w


def _check_grads(name, eng, l1g, q, n):
    g = eng.grads
    floor = 1e-3 * max(np.abs(l1g[q + "grad_" + f]).max() for f in FIELDS)
    for f in FIELDS + ("screen_norms",):
        ok, rel = normwise_ok(getattr(g, f).cpu().numpy().reshape(n, -1),
                              l1g[q + "grad_" + f].reshape(n, -1), floor)
        assert ok, (name, q, f, rel)
    assert np.array_equal(eng.vis.cpu().numpy().astype(bool), l1g[q + "grad_visible"]), (name, q)


def test_train_pair_matches_reference(golden, l1g):
    """gamma = 0: Trainer.step's calls, verbatim - the overlapped forward +
    reverse replay (xg_composite_train_pair) then the chain rule."""
    import torch

    for name in l1g["scenes"]:
        name = str(name)
        cloud, cam, eng, stats, h, w = _scene(golden, name)
        tgt = torch.as_tensor(l1g[name + "/target"], device="cuda").contiguous()
        fr = eng.frame
        fr.preprocess(cloud, cam)
        fr.bin_async()
        fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
        if fr.finish_bin():
            fr.train_pair(tgt, eng.l1, eng.acc, 1.0 / (h * w))
        fr.backward(cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, stats=stats,
                    replay_done=True)
        torch.cuda.synchronize()
        q = name + "/g0.0/"
        value = float(eng.l1.item()) / (h * w)
        ref = float(l1g[q + "loss"])
        assert abs(value - ref) <= 1e-6 * abs(ref), (name, value, ref)
        _check_grads(name, eng, l1g, q, cloud.n_points)


def test_fused_l1_matches_reference(golden, l1g):
    """gamma = 0, the sequential calls: xg_composite_fwd_train's fused L1 sum,
    then xg_composite_bwd's fused sign upstream."""
    import torch

    for name in l1g["scenes"]:
        name = str(name)
        cloud, cam, eng, stats, h, w = _scene(golden, name)
        tgt = torch.as_tensor(l1g[name + "/target"], device="cuda").contiguous()
        fr = eng.frame
        fr.preprocess(cloud, cam)
        fr.bin_async()
        fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        if fr.finish_bin():
            fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        fr.backward(cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, target=tgt,
                    l1_scale=1.0 / (h * w), stats=stats)
        torch.cuda.synchronize()
        q = name + "/g0.0/"
        value = float(eng.l1.item()) / (h * w)
        ref = float(l1g[q + "loss"])
        assert abs(value - ref) <= 1e-6 * abs(ref), (name, value, ref)
        _check_grads(name, eng, l1g, q, cloud.n_points)


def test_fused_l1_ssim_matches_reference(golden, l1g):
    """gamma = 0.2: xg_ssim writes dL/dI = (1-gamma) sign / HW - gamma dSSIM/dI
    into the backward's input (Trainer.step's gamma > 0 branch)."""
    import torch

    from paper_2403_04116_b200.metrics import SsimEngine

    gamma = 0.2
    for name in l1g["scenes"]:
        name = str(name)
        if min(*_scene(golden, name)[4:]) < 11:  # SSIM needs an 11x11 window
            continue
        cloud, cam, eng, stats, h, w = _scene(golden, name)
        tgt = torch.as_tensor(l1g[name + "/target"], device="cuda").contiguous()
        fr = eng.frame
        fr.preprocess(cloud, cam)
        fr.ensure_binned()
        fr.composite(target=tgt, l1_sum=eng.l1, train=True)
        eng.ssim = SsimEngine(h, w, cloud.device)
        s_dev = eng.ssim.run(fr.image, tgt, 1.0, dl=eng.dl, dl_ssim_scale=-gamma,
                             dl_l1_scale=(1.0 - gamma) / (h * w))
        fr.backward(cloud, eng.acc, eng.grads.flat, eng.grads.screen_norms, eng.vis, dl_dimage=eng.dl,
                    stats=stats)
        torch.cuda.synchronize()
        q = f"{name}/g{gamma}/"
        value = (1 - gamma) * float(eng.l1.item()) / (h * w) + gamma * (1 - float(s_dev.item()))
        ref = float(l1g[q + "loss"])
        assert abs(value - ref) <= 1e-6 * abs(ref), (name, value, ref)
        dl_ref = l1g[q + "dl"]
        ok, rel = normwise_ok(eng.dl.cpu().numpy(), dl_ref, 0.0)
        assert ok, (name, "dl", rel)
        _check_grads(name, eng, l1g, q, cloud.n_points)
