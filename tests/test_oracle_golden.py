"""Pin the CPU oracle to the reference's own outputs (tests/golden/golden.npz,
generated from xsplat 0.1.0 by tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise_ok, scene_fields, scene_names
from oracle import oracle as orc

PARAM_FIELDS = orc.PARAM_FIELDS


def cam_of(g, name):
    l_so, l_sd, w, h, pitch, phi = g[name + "/camera"]
    return orc.camera_from_view(l_so, l_sd, int(w), int(h), pitch, phi)


def ref_rects(means2d, radii, w, h):
    """frontend.py:143-147 evaluated on the reference's float64 outputs."""
    ntx, nty = (w + 15) // 16, (h + 15) // 16
    tx0 = np.maximum(np.floor((means2d[:, 0] - radii) / 16), 0)
    tx1 = np.minimum(np.floor((means2d[:, 0] + radii) / 16), ntx - 1)
    ty0 = np.maximum(np.floor((means2d[:, 1] - radii) / 16), 0)
    ty1 = np.minimum(np.floor((means2d[:, 1] + radii) / 16), nty - 1)
    return np.stack([tx0, ty0, tx1, ty1], 1).astype(np.int64)


@pytest.fixture(scope="module")
def oracle_runs(golden):
    out = {}
    for name in scene_names(golden):
        cam = cam_of(golden, name)
        fields = scene_fields(golden, name)
        r = orc.render(fields, golden[name + "/basis_weights"], cam)
        out[name] = (cam, fields, r)
    return out


def test_golden_has_scenes(golden):
    assert len(scene_names(golden)) >= 10


def test_active_set_and_geometry(golden, oracle_runs):
    for name, (cam, _, r) in oracle_runs.items():
        p = name + "/"
        pre = r["pre"]
        act = np.flatnonzero(pre["active"])
        assert np.array_equal(act, golden[p + "active_indices"]), name
        if act.size == 0:
            continue
        for key, mine in (("means2d", pre["mean2d"]), ("radii", pre["radius"]), ("conics", pre["conic"]),
                          ("cov2d", pre["cov2d"]), ("depths", pre["depth"]), ("t_cam", pre["t_cam"])):
            ref = golden[p + key]
            # relative to each row's largest component (off-diagonal conic
            # entries of isotropic splats are rounding noise around 0)
            row = np.abs(ref).reshape(ref.shape[0], -1).max(axis=1)
            row = row.reshape((-1,) + (1,) * (ref.ndim - 1))
            err = np.abs(mine[act] - ref) / np.maximum(row, 1e-300)
            # radii: lambda_max = mid + sqrt(mid^2 - det) cancels for near-isotropic
            # splats even in float64 (frontend.py:139-140), in the reference too
            tol = 1e-7 if key == "radii" else 1e-9
            assert err.max() < tol, (name, key, err.max())
        # float32 intensities / opacities vs float64 reference
        assert np.allclose(pre["inten"][act], golden[p + "intensities"], rtol=2e-7, atol=0), name
        assert np.allclose(pre["opacity"][act], golden[p + "opacities"], rtol=1e-12, atol=0), name


def test_tile_rects_bit_exact(golden, oracle_runs):
    for name, (cam, _, r) in oracle_runs.items():
        p = name + "/"
        act = np.flatnonzero(r["pre"]["active"])
        if act.size == 0:
            continue
        ref = ref_rects(golden[p + "means2d"], golden[p + "radii"], cam.width, cam.height)
        assert np.array_equal(r["pre"]["rect"][act].astype(np.int64), ref), name


def test_entry_order_and_ranges(golden, oracle_runs):
    """Ranges and order bit-exact: the oracle reproduces the reference's
    float64 t_z (same fma order as BLAS) and sorts by it, index tie-break."""
    total_diff = 0
    for name, (cam, _, r) in oracle_runs.items():
        p = name + "/"
        pre, b = r["pre"], r["bin"]
        assert np.array_equal(b["tile_ranges"], golden[p + "tile_ranges"]), name
        act = np.flatnonzero(pre["active"])
        rowmap = np.full(pre["active"].shape[0], -1, np.int64)
        rowmap[act] = np.arange(act.size)
        mine = rowmap[b["entry_splat"].astype(np.int64)]
        ref = golden[p + "entry_splat"].astype(np.int64)
        assert mine.shape == ref.shape, name
        keys = pre["depth_key"][act]
        for t0, t1 in b["tile_ranges"]:
            m, rf = mine[t0:t1], ref[t0:t1]
            assert np.array_equal(np.sort(m), np.sort(rf)), name
            # both orders have non-decreasing float32 keys -> they differ only
            # inside equal-key runs; the oracle breaks those by index
            total_diff += int((m != rf).sum())
    assert total_diff == 0


def test_image_within_1e4_relative(golden, oracle_runs):
    for name, (cam, _, r) in oracle_runs.items():
        ref = golden[name + "/image"]
        img = r["image"].astype(np.float64)
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.all(np.abs(img - ref) <= 1e-4 * np.abs(ref) + 1e-6 * scale), (
            name, np.abs(img - ref).max())


def test_kernel_gradients(golden, oracle_runs):
    for name, (cam, _, r) in oracle_runs.items():
        p = name + "/"
        act = np.flatnonzero(r["pre"]["active"])
        if act.size == 0:
            continue
        kg = orc.composite_bwd(r["pre"], r["bin"], cam.height, cam.width, golden[p + "dl"])
        refs = {k: golden[p + "k_" + k] for k in ("g_mean", "g_conic", "g_int", "g_alpha")}
        floor = 1e-3 * max(np.abs(v).max() for v in refs.values())
        for k, ref in refs.items():
            ok, rel = normwise_ok(kg[k][act], ref, floor)
            assert ok, (name, k, rel)


def test_preprocess_backward(golden, oracle_runs):
    for name, (cam, fields, r) in oracle_runs.items():
        p = name + "/"
        kg = orc.composite_bwd(r["pre"], r["bin"], cam.height, cam.width, golden[p + "dl"])
        g = orc.preprocess_bwd(fields, golden[p + "basis_weights"], cam, r["pre"], kg)
        refs = {f: golden[p + "grad_" + f] for f in PARAM_FIELDS}
        floor = 1e-3 * max(np.abs(v).max() for v in refs.values())
        for f in PARAM_FIELDS:
            ok, rel = normwise_ok(g[f], refs[f], floor)
            assert ok, (name, f, rel)
        assert np.array_equal(g["visible"], golden[p + "grad_visible"]), name
        ok, rel = normwise_ok(g["screen_norms"], golden[p + "grad_screen_norms"], 0.0)
        assert ok, (name, "screen_norms", rel)


def _unflat(vec, n, nf):
    out, o = {}, 0
    for f, wdt in zip(PARAM_FIELDS, (3, 4, 3, 1, nf)):
        out[f] = vec[o:o + n * wdt].reshape(n, wdt) if wdt > 1 or f != "raw_opacities" else vec[o:o + n]
        if f == "raw_opacities":
            out[f] = vec[o:o + n]
        o += n * wdt
    return out


def test_adam_matches_reference(golden):
    n, nf = (int(v) for v in golden["adam/n"])
    params = _unflat(golden["adam/params0"].astype(np.float64), n, nf)
    m = {f: np.zeros_like(v) for f, v in params.items()}
    v = {f: np.zeros_like(x) for f, x in params.items()}
    step = 0
    for s in range(3):
        grads = _unflat(golden[f"adam/grads{s}"], n, nf)
        lr = dict(zip(PARAM_FIELDS, golden[f"adam/lr{s}"]))
        step = orc.adam_step(params, grads, m, v, step, lr)
        ref = _unflat(golden[f"adam/params{s + 1}"], n, nf)
        for f in PARAM_FIELDS:
            assert np.allclose(params[f], ref[f], rtol=1e-12, atol=1e-14), (s, f)


def test_densify_matches_reference(golden):
    p = "densify/"
    params = {f: golden[p + f] for f in PARAM_FIELDS}
    m = {f: golden[p + "m_" + f] for f in PARAM_FIELDS}
    v = {f: golden[p + "v_" + f] for f in PARAM_FIELDS}
    gthr, sthr, pthr, split, cap, seed = golden[p + "cfg"]
    rng = np.random.default_rng(int(seed))
    new, nm, nv, rep = orc.densify(params, m, v, golden[p + "norm_sum"], golden[p + "obs_count"],
                                   golden[p + "world_grad_sum"], gthr, sthr, pthr, split, int(cap),
                                   lambda k: rng.standard_normal((k, 2, 3)))
    assert [rep[k] for k in ("pruned", "cloned", "split", "n_points")] == list(golden[p + "report"])
    for f in PARAM_FIELDS:
        assert np.allclose(new[f], golden[p + "new_" + f], rtol=1e-12, atol=1e-12), f
        assert np.array_equal(nm[f], golden[p + "newm_" + f]), f
        assert np.array_equal(nv[f], golden[p + "newv_" + f]), f
