"""Loss golden vectors from the REAL reference (xsplat 0.1.0): the training
objective the trainer fuses into its kernels (trainer.py:109-123) followed by
render_backward (backward.py:21-124).  Run in the build container:

    python tests/golden/make_golden_l1.py      # -> tests/golden/l1.npz

For scenes of tests/golden/golden.npz (same float32 clouds and cameras), a
target is the reference's own image moved by +-(0.5 .. 1.5) % of its maximum
per pixel (so sign(I - target) is robust to float32-vs-float64 rendering);
for gamma = 0 (the default, L1 only) and gamma = 0.2 (the paper's L1 + SSIM)
the fixture stores the loss value, the pixel gradient and every
RenderGradients field the reference computes from that gradient.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.gaussians import GaussianCloud  # noqa: E402
from xsplat.geometry import ScannerConfig, extrinsic_from_angle, intrinsic_from_config  # noqa: E402
from xsplat.rasterizer import render, render_backward, set_backend  # noqa: E402
from xsplat.trainer import PARAM_FIELDS, loss  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = HERE / "l1.npz"
SCENES = ("rand1", "rand3", "dense", "aniso", "acui20_64_0.7000", "acui36_128_0.7000")


def main():
    set_backend("compiled")
    g = np.load(HERE / "golden.npz")
    rng = np.random.default_rng(4242)
    st: dict = {}
    for name in SCENES:
        p = name + "/"
        f = {k: g[p + k].astype(np.float64) for k in PARAM_FIELDS}
        cloud = GaussianCloud(*(f[k] for k in PARAM_FIELDS), g[p + "basis_weights"].astype(np.float64))
        l_so, l_sd, w, h, pitch, phi = g[p + "camera"]
        sc = ScannerConfig(l_so, l_sd, int(w), int(h), pitch)
        proj, sp = render(cloud, extrinsic_from_angle(sc, phi), intrinsic_from_config(sc), (int(h), int(w)))
        img = proj.pixels
        s = 0.01 * max(float(np.abs(img).max()), 1e-3)
        sgn = np.where(rng.uniform(size=img.shape) < 0.5, -1.0, 1.0)
        target = np.asarray(img + s * sgn * (0.5 + rng.uniform(size=img.shape)), np.float32)
        st[p + "target"] = target
        for gamma in (0.0, 0.2):
            q = f"{p}g{gamma}/"
            value, dl = loss(proj, target.astype(np.float64), gamma)
            grads = render_backward(cloud, sp, dl)
            st[q + "loss"] = np.array(value)
            st[q + "dl"] = dl
            for k in PARAM_FIELDS + ("screen_norms", "visible"):
                st[q + "grad_" + k] = np.asarray(getattr(grads, k))
    st["scenes"] = np.array(SCENES)
    np.savez_compressed(OUT, **st)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
