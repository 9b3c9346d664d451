"""Golden vectors for the phantom projector and dataset pipeline from the
REAL reference (xsplat 0.1.0 phantom.py:117-250, dataset.py:66-115), built
into oracle/_ref by oracle/build_ref.sh.  Run in the build container:

    python tests/golden/make_golden_phantom.py     # -> tests/golden/phantom.npz
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.dataset import add_noise, make_projection_set  # noqa: E402
from xsplat.geometry import ScannerConfig, equal_interval_angles  # noqa: E402
from xsplat.phantom import (  # noqa: E402
    Cuboid,
    Ellipsoid,
    default_phantom_primitives,
    make_phantom,
    project_phantom,
)

OUT = Path(__file__).resolve().parent / "phantom.npz"


def main():
    st = {}
    # A: small anisotropic volume, non-square detector, 4 angles, full pipeline
    grid, vs = (24, 20, 28), np.array([8.0 / 3.0, 3.2, 16.0 / 7.0])
    prims = default_phantom_primitives(np.array(grid) * vs)
    ph = make_phantom(prims, grid, vs)
    sc = ScannerConfig(1000.0, 1500.0, 48, 40, 6.0, equal_interval_angles(4))
    st["A/grid"], st["A/voxel_size"] = np.array(grid), vs
    st["A/densities"] = ph.densities
    st["A/scanner"] = np.array([1000.0, 1500.0, 48, 40, 6.0, 4])
    ps = make_projection_set(ph, sc)
    st["A/raw"] = np.stack([project_phantom(ph, sc, float(p)) for p in sc.angles])
    st["A/images"], st["A/normalization"] = ps.images, np.float64(ps.normalization)
    noisy = add_noise(ps, 0.03, 0)
    st["A/noisy"] = noisy.images
    st["A/raw_step05"] = project_phantom(ph, sc, 0.7, step_factor=0.5)
    # B: the C2 phantom (88^3 lattice span, 200 mm) at 128^2, one view
    g = 88
    vsb = np.full(3, 200.0 / g)
    phb = make_phantom(default_phantom_primitives(np.full(3, 200.0)), (g, g, g), vsb)
    scb = ScannerConfig(1000.0, 1500.0, 128, 128, 192.0 / 128, np.array([0.3]))
    st["B/g"] = np.int64(g)
    st["B/density_sum"] = np.float64(phb.densities.sum())
    st["B/density_nnz"] = np.int64((phb.densities > 0).sum())
    st["B/raw"] = project_phantom(phb, scb, 0.3)
    # C: primitives touching the volume faces (edge samples, zero-density rays)
    grid_c, vsc = (16, 16, 16), np.full(3, 2.0)
    phc = make_phantom([Cuboid([0.0, 0.0, 0.0], [16.0, 16.0, 16.0], 0.5),
                        Ellipsoid([8.0, -8.0, 0.0], [8.0, 8.0, 8.0], 0.25)], grid_c, vsc)
    scc = ScannerConfig(1000.0, 1500.0, 32, 32, 3.0, np.array([0.0, np.pi / 4]))
    st["C/densities"] = phc.densities
    st["C/raw"] = np.stack([project_phantom(phc, scc, float(p)) for p in scc.angles])
    np.savez_compressed(OUT, **st)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
