"""GPU parity: the CUDA engine (through the package API / C ABI) against the
CPU oracle (bit-exact integers) and the reference's golden outputs (1e-4)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise_ok, scene_fields, scene_names
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

PARAM_FIELDS = orc.PARAM_FIELDS


@pytest.fixture(scope="module")
def xg():
    import torch

    import paper_2403_04116_b200 as xg

    torch.cuda.set_device(0)
    return xg


def _scene(golden, name, xg):
    import torch

    p = name + "/"
    fields = scene_fields(golden, name)
    cloud = xg.GaussianCloud(**fields, basis_weights=golden[p + "basis_weights"], device="cuda")
    l_so, l_sd, w, h, pitch, phi = golden[p + "camera"]
    sc = xg.ScannerConfig(l_so, l_sd, int(w), int(h), pitch)
    ext = xg.extrinsic_from_angle(sc, phi)
    intr = xg.intrinsic_from_config(sc)
    cam = orc.camera_from_view(l_so, l_sd, int(w), int(h), pitch, phi)
    ref = orc.render(fields, golden[p + "basis_weights"], cam)
    proj, splats = xg.render(cloud, ext, intr, (int(h), int(w)))
    torch.cuda.synchronize()
    return cloud, proj, splats, ref, cam


@pytest.fixture(scope="module")
def runs(golden, xg):
    return {name: _scene(golden, name, xg) for name in scene_names(golden)}


def test_projection_bit_exact(golden, runs):
    for name, (cloud, proj, sp, ref, cam) in runs.items():
        pre = ref["pre"]
        act = np.flatnonzero(pre["active"])
        assert np.array_equal(sp.active_indices.cpu().numpy(), act), name
        assert np.array_equal(act, golden[name + "/active_indices"]), name
        if act.size == 0:
            continue
        rect = sp.frame.rect.cpu().numpy().astype(np.int64) & 0xFFFF
        assert np.array_equal(rect[act], pre["rect"][act]), name
        # float64 geometry: bit-identical to the oracle (same op order)
        assert np.array_equal(sp.radii.cpu().numpy(), pre["radius"][act]), name
        assert np.array_equal(sp.means2d.cpu().numpy(), pre["mean2d"][act]), name
        assert np.array_equal(sp.conics.cpu().numpy(), pre["conic"][act]), name
        assert np.array_equal(sp.depths.cpu().numpy(), pre["depth"][act]), name
        assert np.array_equal(sp.intensities.cpu().numpy(), pre["inten"][act]), name
        assert np.array_equal(sp.frame.coef.cpu().numpy()[act], pre["coef"][act]), name


def test_binning_bit_exact(golden, runs):
    for name, (cloud, proj, sp, ref, cam) in runs.items():
        assert np.array_equal(sp.tile_ranges.cpu().numpy(), ref["bin"]["tile_ranges"]), name
        assert np.array_equal(sp.tile_ranges.cpu().numpy(), golden[name + "/tile_ranges"]), name
        assert np.array_equal(sp.entry_ids.cpu().numpy().astype(np.uint32), ref["bin"]["entry_splat"]), name
        # reference's active-row form, against the real reference
        assert np.array_equal(sp.entry_splat.cpu().numpy(), golden[name + "/entry_splat"]), name


def test_contributor_counts(golden, runs):
    total_amb = 0
    for name, (cloud, proj, sp, ref, cam) in runs.items():
        amb = ref["ambiguous"].astype(bool)
        total_amb += int(amb.sum())
        nc = sp.frame.n_contrib.cpu().numpy()
        assert np.array_equal(nc[~amb], ref["n_contrib"][~amb]), (name, int((nc != ref["n_contrib"]).sum()))
    assert total_amb < 50


def test_image_parity(golden, runs):
    for name, (cloud, proj, sp, ref, cam) in runs.items():
        img = proj.pixels.cpu().numpy().astype(np.float64)
        gold = golden[name + "/image"]
        scale = max(np.abs(gold).max(), 1e-30)
        assert np.all(np.abs(img - gold) <= 1e-4 * np.abs(gold) + 1e-6 * scale), (name, np.abs(img - gold).max())
        # against the float32 oracle: only MUFU.EX2 vs exp2 rounding differs
        o = ref["image"].astype(np.float64)
        assert np.all(np.abs(img - o) <= 2e-5 * np.abs(o) + 1e-7 * scale), (name, np.abs(img - o).max())
        tf = sp.frame.t_final.cpu().numpy()
        assert np.allclose(tf, ref["t_final"], rtol=1e-4, atol=1e-7), name


@pytest.mark.parametrize("batch", [1, 2])
def test_image_only_parity(golden, xg, batch):
    """Image-only launches (sweep renderer / evaluate: speculative test-free
    batches, re-run exactly where a pixel crosses the transmittance floor)
    against the reference's golden images and the float32 oracle."""
    from paper_2403_04116_b200.inference import SweepRenderer

    for name in scene_names(golden):
        p = name + "/"
        fields = scene_fields(golden, name)
        cloud = xg.GaussianCloud(**fields, basis_weights=golden[p + "basis_weights"], device="cuda")
        l_so, l_sd, w, h, pitch, phi = golden[p + "camera"]
        sc = xg.ScannerConfig(l_so, l_sd, int(w), int(h), pitch)
        img = SweepRenderer(cloud, sc, batch=batch).render(np.array([phi] * batch))
        cam = orc.camera_from_view(l_so, l_sd, int(w), int(h), pitch, phi)
        o = orc.render(fields, golden[p + "basis_weights"], cam)["image"].astype(np.float64)
        gold = golden[p + "image"]
        scale = max(np.abs(gold).max(), 1e-30)
        for v in img.cpu().numpy().astype(np.float64):
            assert np.all(np.abs(v - gold) <= 1e-4 * np.abs(gold) + 1e-6 * scale), (name, np.abs(v - gold).max())
            assert np.all(np.abs(v - o) <= 2e-5 * np.abs(o) + 1e-7 * scale), (name, np.abs(v - o).max())


def test_backward_parity(golden, runs, xg):
    import torch

    for name, (cloud, proj, sp, ref, cam) in runs.items():
        p = name + "/"
        n = cloud.n_points
        kg = {k: torch.zeros(s, dtype=torch.float64, device="cuda")
              for k, s in (("g_mean", (n, 2)), ("g_conic", (n, 3)), ("g_int", n), ("g_alpha", n))}
        grads = xg.render_backward(cloud, sp, torch.as_tensor(golden[p + "dl"]), kernel_grads=kg)
        torch.cuda.synchronize()
        act = np.flatnonzero(ref["pre"]["active"])
        if act.size:
            refs = {k: golden[p + "k_" + k] for k in ("g_mean", "g_conic", "g_int", "g_alpha")}
            floor = 1e-3 * max(np.abs(v).max() for v in refs.values())
            for k, want in refs.items():
                ok, rel = normwise_ok(kg[k].cpu().numpy()[act], want, floor)
                assert ok, (name, "kernel", k, rel)
        refs = {f: golden[p + "grad_" + f] for f in PARAM_FIELDS}
        floor = 1e-3 * max(np.abs(v).max() for v in refs.values())
        for f in PARAM_FIELDS:
            ok, rel = normwise_ok(getattr(grads, f).cpu().numpy(), refs[f], floor)
            assert ok, (name, f, rel)
        assert np.array_equal(grads.visible.cpu().numpy(), golden[p + "grad_visible"]), name
        ok, rel = normwise_ok(grads.screen_norms.cpu().numpy(), golden[p + "grad_screen_norms"], 0.0)
        assert ok, (name, "screen_norms", rel)


def test_training_forward(golden, runs, xg):
    """The trainer's forward (xg_composite_fwd_train): image / t_final equal
    the exact tracking forward to float32 rounding; n_contrib is the exact
    count for terminated pixels and the tile length for the rest; the reverse
    replay from it gives the reference's gradients."""
    import torch

    n_term = 0
    for name, (cloud, proj, sp, ref, cam) in runs.items():
        p = name + "/"
        fr = sp.frame
        if sp.n_active == 0:
            continue
        fr.composite()  # exact tracking forward (render()'s)
        img0, tf0, nc0 = fr.image.clone(), fr.t_final.clone(), fr.n_contrib.clone()
        fr.composite(train=True)
        torch.cuda.synchronize()
        scale = float(img0.abs().max())
        assert bool(((fr.image - img0).abs() <= 2e-5 * img0.abs() + 1e-7 * scale).all()), name
        assert bool(((fr.t_final - tf0).abs() <= 2e-5 * tf0.abs() + 1e-9).all()), name
        term = tf0 < 1e-4
        n_term += int(term.sum())
        assert torch.equal(fr.n_contrib[term], nc0[term]), name
        h, w = fr.h, fr.w
        ntx = (w + 15) // 16
        yy, xx = torch.meshgrid(torch.arange(h, device="cuda"), torch.arange(w, device="cuda"), indexing="ij")
        rng = sp.tile_ranges[(yy // 16) * ntx + xx // 16]
        length = (rng[..., 1] - rng[..., 0]).to(torch.int32)
        assert torch.equal(fr.n_contrib[~term], length[~term]), name
        assert bool((fr.n_contrib >= nc0).all()), name
        n = cloud.n_points
        kg = {k: torch.zeros(s_, dtype=torch.float64, device="cuda")
              for k, s_ in (("g_mean", (n, 2)), ("g_conic", (n, 3)), ("g_int", n), ("g_alpha", n))}
        xg.render_backward(cloud, sp, torch.as_tensor(golden[p + "dl"]), kernel_grads=kg)
        torch.cuda.synchronize()
        act = np.flatnonzero(ref["pre"]["active"])
        refs = {k: golden[p + "k_" + k] for k in ("g_mean", "g_conic", "g_int", "g_alpha")}
        floor = 1e-3 * max(np.abs(v).max() for v in refs.values())
        for k, want in refs.items():
            ok, rel = normwise_ok(kg[k].cpu().numpy()[act], want, floor)
            assert ok, (name, k, rel)
        fr.composite()  # leave the exact forward for the other tests
    assert n_term > 0  # the golden set has terminating pixels


def test_plugin_forward_backward_tiles(golden, xg):
    """The reference's kernel-backend contract served by xg_forward_tiles /
    xg_backward_tiles, fed the reference's own SplatList arrays."""
    from paper_2403_04116_b200.rasterizer import get_kernels

    k = get_kernels()
    for name in scene_names(golden):
        p = name + "/"
        if golden[p + "active_indices"].size == 0:
            continue
        _, _, w, h, _, _ = golden[p + "camera"]
        args = [golden[p + a] for a in ("means2d", "conics", "intensities", "opacities", "entry_splat",
                                        "tile_ranges")]
        img = k.forward_tiles(int(h), int(w), *args).cpu().numpy()
        gold = golden[p + "image"]
        scale = max(np.abs(gold).max(), 1e-30)
        assert np.all(np.abs(img - gold) <= 1e-4 * np.abs(gold) + 1e-6 * scale), name
        gm, gc, gi, ga = (t.cpu().numpy() for t in k.backward_tiles(int(h), int(w), *args, golden[p + "dl"]))
        refs = {"g_mean": gm, "g_conic": gc, "g_int": gi, "g_alpha": ga}
        floor = 1e-3 * max(np.abs(golden[p + "k_" + kk]).max() for kk in refs)
        for kk, mine in refs.items():
            ok, rel = normwise_ok(mine, golden[p + "k_" + kk], floor)
            assert ok, (name, kk, rel)
