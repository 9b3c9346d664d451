"""Training-trajectory golden vectors from the REAL reference (xsplat 0.1.0
``train``, trainer.py:330-438).  Run in the build container:

    python tests/golden/make_golden_train.py     # -> tests/golden/train.npz

Two short runs through the whole loop - view permutation, render, loss,
render_backward, DensifyStats, Adam with the decaying position LR, density
control (two events), logging and held-out evaluation:

* ``l1``: gamma = 0 (the default objective);
* ``ssim_reset``: gamma = 0.2 (L1 + SSIM, the paper's) with an opacity reset.

Dataset: the reference pipeline (default phantom voxelised on a 32^3 grid of
the 100 mm cube, cone-beam projected, normalised, 3 % noise seed 0) at 32^2,
pitch 6, 20 views; stored in the fixture so the engine trains on the same
float32 targets.  Initial cloud: ACUI cuboid (grid 32, interval 4: 1,331
Gaussians), rounded to float32.  Stored: the metrics rows, the checkpoint
at iteration 250 (between the two density-control events) and the final
cloud."""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.acui import CuboidSpec, init_alternative  # noqa: E402
from xsplat.cloudio import load_cloud  # noqa: E402
from xsplat.dataset import add_noise, make_projection_set  # noqa: E402
from xsplat.gaussians import GaussianCloud  # noqa: E402
from xsplat.geometry import ScannerConfig, equal_interval_angles  # noqa: E402
from xsplat.phantom import default_phantom_primitives, make_phantom  # noqa: E402
from xsplat.rasterizer import set_backend  # noqa: E402
from xsplat.trainer import PARAM_FIELDS, TrainConfig, train  # noqa: E402

OUT = Path(__file__).resolve().parent / "train.npz"
CASES = {
    "l1": dict(gamma=0.0, opacity_reset_interval=0),
    "ssim_reset": dict(gamma=0.2, opacity_reset_interval=150),
}
ROW_KEYS = ("iteration", "loss", "train_psnr", "test_psnr", "test_ssim", "n_points")


def main():
    set_backend("compiled")
    sc = ScannerConfig(1000.0, 1500.0, 32, 32, 6.0, equal_interval_angles(20))
    extent = np.full(3, 100.0)
    ph = make_phantom(default_phantom_primitives(tuple(extent)), (32, 32, 32), extent / 32)
    ds = add_noise(make_projection_set(ph, sc), 0.03, 0)
    c = init_alternative("cuboid", CuboidSpec(extent=(100.0,) * 3, grid=(32,) * 3, interval=4), 16, 0)
    f32 = {k: np.asarray(getattr(c, k), np.float32) for k in PARAM_FIELDS}
    cloud = GaussianCloud(*(f32[k].astype(np.float64) for k in PARAM_FIELDS), np.ones(16))
    st = {"images": ds.images, "clean_images": ds.clean_images, "train_indices": ds.train_indices,
          "test_indices": ds.test_indices, "scanner": np.array([1000.0, 1500.0, 32, 32, 6.0, 20])}
    for k in PARAM_FIELDS:
        st["init/" + k] = f32[k]
    for name, kw in CASES.items():
        cfg = TrainConfig(iterations=300, densify_from_iter=100, densify_interval=100, densify_until_iter=300,
                          log_interval=10, eval_interval=100, checkpoint_iterations=(250,), **kw)
        with tempfile.TemporaryDirectory() as tmp:
            res = train(ds, cloud, cfg, out_dir=tmp)
            ck = load_cloud(Path(tmp) / "ckpt_000250.ply")
        for k in PARAM_FIELDS:
            st[name + "/ckpt250_" + k] = np.asarray(getattr(ck, k))
        rows = np.array([[np.nan if r[k] is None else float(r[k]) for k in ROW_KEYS] for r in res.metrics])
        st[name + "/rows"] = rows
        for k in PARAM_FIELDS:
            st[name + "/final_" + k] = np.asarray(getattr(res.cloud, k))
        st[name + "/cfg"] = np.array([cfg.gamma, cfg.opacity_reset_interval])
        print(name, rows[-1], res.cloud.n_points)
    np.savez_compressed(OUT, **st)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
