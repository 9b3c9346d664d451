"""A checkpoint written by the REAL reference (xsplat cloudio.py:31-57) for
the PLY interchange test.  Run in the build container:

    python tests/golden/make_golden_cloudio.py     # -> tests/golden/ref_cloud.ply
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.cloudio import save_cloud  # noqa: E402
from xsplat.gaussians import GaussianCloud  # noqa: E402

rng = np.random.default_rng(7)
n, nf = 40, 5
f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
q = rng.normal(size=(n, 4))
cloud = GaussianCloud(f32(rng.uniform(-40, 40, (n, 3))), f32(q / np.linalg.norm(q, axis=1, keepdims=True)),
                      f32(np.log(rng.uniform(2, 9, (n, 3)))), f32(rng.normal(size=n)),
                      f32(rng.normal(scale=0.3, size=(n, nf))), f32(rng.uniform(0.5, 1.5, nf)))
save_cloud(cloud, Path(__file__).resolve().parent / "ref_cloud.ply")
print("wrote ref_cloud.ply")
