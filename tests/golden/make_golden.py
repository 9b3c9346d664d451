"""Generate golden vectors from the REAL reference (xsplat 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py          # uses oracle/_ref (oracle/build_ref.sh)

Every scene's parameters are rounded to float32 first, so the float64
reference and the float32-parameter engine see identical inputs.  Stored
per scene (``<scene>/<key>`` in golden.npz):

* inputs: the five cloud fields, basis weights, camera (L_SO, L_SD, W, H,
  pitch, phi), upstream pixel gradient ``dl``;
* reference outputs: image (float64), SplatList fields (active_indices,
  means2d, conics, cov2d, radii, depths, entry_splat, tile_ranges),
  kernel-level gradients (backward_tiles) and RenderGradients fields.

Plus fixtures for Adam and density control (trainer.py:147-268).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(REF))

from xsplat.acui import CuboidSpec, init_alternative  # noqa: E402
from xsplat.gaussians import GaussianCloud, logit  # noqa: E402
from xsplat.geometry import ScannerConfig, extrinsic_from_angle, intrinsic_from_config  # noqa: E402
from xsplat.rasterizer import get_kernels, render, render_backward, set_backend  # noqa: E402
from xsplat.trainer import (  # noqa: E402
    PARAM_FIELDS,
    DensifyStats,
    OptimizerState,
    TrainConfig,
    adam_step,
    densify_and_prune,
)
from xsplat.rasterizer import RenderGradients  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"


def f32_cloud(cloud: GaussianCloud) -> GaussianCloud:
    f = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    return GaussianCloud(f(cloud.positions), f(cloud.rotations), f(cloud.log_scales), f(cloud.raw_opacities),
                         f(cloud.features), f(cloud.basis_weights))


def random_cloud(n, rng, n_features=4, pos_scale=40.0, scale_range=(3.0, 10.0), opacity_range=(0.05, 0.5),
                 basis_weights=None):
    # conftest.py:19-40 of the reference
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    alphas = rng.uniform(*opacity_range, size=n)
    return GaussianCloud(
        positions=rng.uniform(-pos_scale, pos_scale, size=(n, 3)),
        rotations=q,
        log_scales=np.log(rng.uniform(*scale_range, size=(n, 3))),
        raw_opacities=np.log(alphas) - np.log1p(-alphas),
        features=rng.normal(scale=0.5, size=(n, n_features)),
        basis_weights=basis_weights,
    )


def scene(store: dict, name: str, cloud: GaussianCloud, l_so, l_sd, w, h, pitch, phi, rng):
    cloud = f32_cloud(cloud)
    sc = ScannerConfig(l_so, l_sd, w, h, pitch)
    ext = extrinsic_from_angle(sc, phi)
    intr = intrinsic_from_config(sc)
    proj, sp = render(cloud, ext, intr, (h, w))
    dl = rng.normal(size=(h, w)) / (h * w)
    grads = render_backward(cloud, sp, dl)
    p = name + "/"
    for f in PARAM_FIELDS:
        store[p + f] = np.asarray(getattr(cloud, f), dtype=np.float32)
    store[p + "basis_weights"] = np.asarray(cloud.basis_weights, dtype=np.float32)
    store[p + "camera"] = np.array([l_so, l_sd, w, h, pitch, phi], dtype=np.float64)
    store[p + "dl"] = dl
    store[p + "image"] = proj.pixels
    for k in ("active_indices", "means2d", "conics", "cov2d", "radii", "depths", "intensities", "opacities",
              "entry_splat", "tile_ranges", "t_cam"):
        store[p + k] = np.asarray(getattr(sp, k))
    if sp.n_active:
        gm, gc, gi, ga = get_kernels().backward_tiles(h, w, sp.means2d, sp.conics, sp.intensities, sp.opacities,
                                                      sp.entry_splat, sp.tile_ranges, dl)
    else:
        gm, gc, gi, ga = (np.zeros((0, 2)), np.zeros((0, 3)), np.zeros(0), np.zeros(0))
    store[p + "k_g_mean"], store[p + "k_g_conic"], store[p + "k_g_int"], store[p + "k_g_alpha"] = gm, gc, gi, ga
    for f in PARAM_FIELDS + ("screen_norms", "visible"):
        store[p + "grad_" + f] = np.asarray(getattr(grads, f))
    return name


def adam_fixture(store: dict, rng):
    cloud = f32_cloud(random_cloud(6, rng, n_features=3))
    state = OptimizerState(cloud)
    cfg = TrainConfig()
    store["adam/params0"] = np.concatenate([np.asarray(getattr(cloud, f)).reshape(-1) for f in PARAM_FIELDS])
    seq = []
    for step in range(3):
        gr = {f: np.asarray(rng.normal(size=getattr(cloud, f).shape), dtype=np.float32).astype(np.float64)
              for f in PARAM_FIELDS}
        g = RenderGradients(**gr, screen_norms=np.zeros(6), visible=np.ones(6, bool))
        lr = {"positions": 1.9e-4 * (0.5 ** step), "rotations": 1e-3, "log_scales": 5e-3, "raw_opacities": 8e-3,
              "features": 2e-3}
        adam_step(cloud, g, state, lr, cfg)
        seq.append((gr, lr))
        store[f"adam/grads{step}"] = np.concatenate([gr[f].reshape(-1) for f in PARAM_FIELDS])
        store[f"adam/lr{step}"] = np.array([lr[f] for f in PARAM_FIELDS])
        store[f"adam/params{step + 1}"] = np.concatenate([np.asarray(getattr(cloud, f)).reshape(-1)
                                                          for f in PARAM_FIELDS])
        store[f"adam/m{step + 1}"] = np.concatenate([state.exp_avg[f].reshape(-1) for f in PARAM_FIELDS])
        store[f"adam/v{step + 1}"] = np.concatenate([state.exp_avg_sq[f].reshape(-1) for f in PARAM_FIELDS])
    store["adam/n"] = np.array([6, 3])


def densify_fixture(store: dict, rng):
    # trainer test fixture (test_trainer.py:172-193) plus a random one
    n = 40
    cloud = f32_cloud(random_cloud(n, rng, n_features=2, scale_range=(0.5, 20.0), opacity_range=(0.001, 0.9)))
    q = np.asarray(cloud.rotations)
    state = OptimizerState(cloud)
    state.step = 9
    for f in PARAM_FIELDS:
        state.exp_avg[f][:] = np.asarray(rng.normal(size=state.exp_avg[f].shape), np.float32)
        state.exp_avg_sq[f][:] = np.asarray(rng.uniform(size=state.exp_avg_sq[f].shape), np.float32)
    stats = DensifyStats.zeros(n)
    stats.norm_sum[:] = np.asarray(rng.uniform(0, 2e-4, size=n), np.float32)
    stats.obs_count[:] = rng.integers(0, 5, size=n)
    stats.world_grad_sum[:] = np.asarray(rng.normal(size=(n, 3)), np.float32)
    cfg = TrainConfig(densify_grad_threshold=2e-5)
    new_cloud, new_state, report = densify_and_prune(cloud, state, stats, cfg, 5.0, np.random.default_rng(77))
    p = "densify/"
    for f in PARAM_FIELDS:
        store[p + f] = np.asarray(getattr(cloud, f), np.float32)
        store[p + "m_" + f] = np.asarray(state.exp_avg[f], np.float32)
        store[p + "v_" + f] = np.asarray(state.exp_avg_sq[f], np.float32)
        store[p + "new_" + f] = np.asarray(getattr(new_cloud, f))
        store[p + "newm_" + f] = np.asarray(new_state.exp_avg[f])
        store[p + "newv_" + f] = np.asarray(new_state.exp_avg_sq[f])
    store[p + "norm_sum"] = stats.norm_sum
    store[p + "obs_count"] = stats.obs_count
    store[p + "world_grad_sum"] = stats.world_grad_sum
    store[p + "report"] = np.array([report["pruned"], report["cloned"], report["split"], report["n_points"]])
    store[p + "cfg"] = np.array([2e-5, 5.0, 0.005, 1.6, 500000, 77])
    del q


def main():
    set_backend("compiled")
    rng = np.random.default_rng(1234)
    store: dict = {}
    names = []
    # conftest-style random scenes (test_rasterizer.py / test_gradients.py sizes)
    for k in range(6):
        n = int(rng.integers(1, 40))
        names.append(scene(store, f"rand{k}", random_cloud(n, rng, scale_range=(2.0, 15.0),
                                                         opacity_range=(0.05, 0.9)),
                           1000.0, 1500.0, 64, 64, 3.0, float(rng.uniform(0, np.pi)), rng))
    names.append(scene(store, "dense", random_cloud(50, rng, pos_scale=20.0, scale_range=(10.0, 30.0),
                                                    opacity_range=(0.6, 0.95)),
                       1000.0, 1500.0, 48, 48, 4.0, 1.1, rng))
    names.append(scene(store, "small16", random_cloud(8, rng, pos_scale=35.0, scale_range=(4.0, 14.0)),
                       1000.0, 1500.0, 16, 16, 12.0, 0.85, rng))
    names.append(scene(store, "aniso", random_cloud(12, rng, n_features=6, scale_range=(1.5, 25.0),
                                                    basis_weights=rng.normal(size=6)),
                       1000.0, 1500.0, 40, 24, 5.0, 0.3, rng))
    # ACUI cuboid lattices on the benchmark geometry (pitch 192/D)
    for g, d, phi in ((20, 64, 0.0), (20, 64, np.pi / 4), (20, 64, 0.7), (36, 128, 0.7)):
        cloud = init_alternative("cuboid", CuboidSpec((100.0,) * 3, (g,) * 3, 2), 16, 0)
        names.append(scene(store, f"acui{g}_{d}_{phi:.4f}", cloud, 1000.0, 1500.0, d, d, 192.0 / d, phi, rng))
    adam_fixture(store, rng)
    densify_fixture(store, rng)
    store["scenes"] = np.array(names)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB): {names}")


if __name__ == "__main__":
    main()
