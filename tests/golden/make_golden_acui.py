"""ACUI initialisation golden vectors from the REAL reference (xsplat
acui.py:60-182).  Run in the build container:

    python tests/golden/make_golden_acui.py     # -> tests/golden/acui.npz
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.acui import CuboidSpec, init_alternative  # noqa: E402

OUT = Path(__file__).resolve().parent / "acui.npz"
CASES = {
    "cuboid": ("cuboid", (100.0, 100.0, 100.0), (20, 20, 20), 2, 4, 0, None, None),
    "cuboid_aniso": ("cuboid", (60.0, 90.0, 120.0), (24, 18, 30), 3, 3, 5, None, None),
    "random": ("random", (100.0, 80.0, 60.0), (16, 16, 16), 2, 4, 1, 300, None),
    "spherical": ("spherical", (100.0, 100.0, 100.0), (16, 16, 16), 2, 5, 2, 250, 40.0),
    "spherical_default": ("spherical", (50.0, 70.0, 90.0), (12, 12, 12), 2, 2, 3, None, None),
}
FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")


def main():
    st = {}
    for name, (strategy, extent, grid, interval, nf, seed, n_points, radius) in CASES.items():
        c = init_alternative(strategy, CuboidSpec(extent=extent, grid=grid, interval=interval), nf, seed,
                             n_points=n_points, radius=radius)
        for f in FIELDS:
            st[f"{name}/{f}"] = getattr(c, f)
    np.savez_compressed(OUT, **st)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
