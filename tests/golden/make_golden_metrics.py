"""Golden vectors for the SSIM / PSNR / loss path from the REAL reference
(xsplat 0.1.0 metrics.py:36-124, trainer.py:109-123), built into oracle/_ref
by oracle/build_ref.sh.  Run in the build container:

    python tests/golden/make_golden_metrics.py     # -> tests/golden/metrics.npz

Images are float32-representable (the engine renders float32), so both
sides see identical inputs; the reference computes in float64.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.metrics import psnr, ssim, ssim_and_gradient  # noqa: E402
from xsplat.trainer import loss  # noqa: E402

OUT = Path(__file__).resolve().parent / "metrics.npz"


def f32(a):
    return np.asarray(a, dtype=np.float32)


def cases(rng):
    a = rng.uniform(size=(64, 64))
    yield "noise64", f32(a), f32(np.clip(a + rng.normal(scale=0.1, size=a.shape), 0, 1)), 1.0
    yy, xx = np.mgrid[0:32, 0:32] / 31.0
    yield ("structured32", f32(0.5 + 0.4 * np.sin(6 * xx) * np.cos(4 * yy)),
           f32(0.5 + 0.4 * np.sin(6 * xx + 0.2) * np.cos(4 * yy)), 1.0)
    yield "ragged13x17", f32(rng.uniform(size=(13, 17))), f32(rng.uniform(size=(13, 17))), 1.0
    yield "range2", f32(2 * rng.uniform(size=(40, 45))), f32(2 * rng.uniform(size=(40, 45))), 2.0
    # detector-sized projection-like pair: smooth blobs, one slightly shifted
    yy, xx = np.mgrid[0:512, 0:512] / 511.0
    img = np.zeros((512, 512))
    for _ in range(12):
        cx, cy, s, amp = rng.uniform(0.2, 0.8), rng.uniform(0.2, 0.8), rng.uniform(0.03, 0.2), rng.uniform(0.1, 0.4)
        img += amp * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
    shifted = np.roll(img, (2, -1), axis=(0, 1)) * 0.97 + 0.01 * rng.normal(size=img.shape)
    yield "proj512", f32(img), f32(shifted), 1.0
    yield "identical", f32(img[:48, :48]), f32(img[:48, :48]), 1.0


def main():
    rng = np.random.default_rng(2403)
    store = {}
    names = []
    for name, a, b, dr in cases(rng):
        names.append(name)
        p = name + "/"
        store[p + "pred"], store[p + "ref"] = a, b
        store[p + "data_range"] = np.float64(dr)
        A, B = a.astype(np.float64), b.astype(np.float64)
        store[p + "ssim"] = np.float64(ssim(A, B, data_range=dr))
        s, g = ssim_and_gradient(A, B, data_range=dr)
        store[p + "ssim_grad"] = g
        store[p + "psnr"] = np.float64(psnr(A, B, data_range=dr))
        if dr == 1.0 and a.size <= 64 * 64:  # (keeps the fixture small)
            for gamma in (0.0, 0.2, 1.0):
                v, dl = loss(A, B, gamma)
                store[p + f"loss_{gamma}"] = np.float64(v)
                store[p + f"loss_grad_{gamma}"] = dl
    store["cases"] = np.array(names)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({len(names)} cases)")


if __name__ == "__main__":
    main()
