"""BLAS accumulation-order guard (CPU).

The engine's float64 camera-space positions reproduce the rounding of the
reference's ``t_cam = positions @ rot_w.T + ext.m[:3, 3]``
(rasterizer/frontend.py:116) as OpenBLAS dgemm computes it in the golden
container: ``fma(w2, z, fma(w1, y, w0 * x)) + t`` (csrc/xg_preprocess.cu).
That is what makes the depth order bit-identical to the reference at exact
real-arithmetic ties (the symmetric phi = pi/4 lattice view).  A different
BLAS micro-kernel (another ISA dispatch, another library) may round
differently; this test fails loudly when the numpy running here departs
from the engine's order, so a golden regenerated on such a host is not
silently trusted.  The producing host of tests/golden/fullsize.npz is in
its ``host`` key."""

from __future__ import annotations

import numpy as np

import fullsize_golden as fg
from oracle import oracle as orc
from paper_2403_04116_b200.geometry import ScannerConfig, extrinsic_from_angle


def blas_order_matches(positions: np.ndarray, phi: float, l_so=1000.0, l_sd=1500.0, d=512) -> tuple[bool, int]:
    sc = ScannerConfig(l_so, l_sd, d, d, 192.0 / d)
    ext = extrinsic_from_angle(sc, phi)
    rot_w = np.asarray(ext.rotation, np.float64)
    pos = np.ascontiguousarray(positions, np.float64)
    numpy_t = pos @ rot_w.T + np.asarray(ext.m, np.float64)[:3, 3]  # frontend.py:116
    cam = orc.camera_from_view(l_so, l_sd, d, d, 192.0 / d, phi)
    n = pos.shape[0]
    fields = {"positions": pos.astype(np.float32), "rotations": np.tile([1.0, 0, 0, 0], (n, 1)),
              "log_scales": np.zeros((n, 3)), "raw_opacities": np.zeros(n), "features": np.zeros((n, 1))}
    pre = orc.preprocess(fields, np.ones(1, np.float32), cam)
    act = pre["active"]  # the oracle writes t_cam for splats that survive every cull
    assert act.sum() > 0.9 * n
    mism = int(np.count_nonzero(np.any(numpy_t[act] != pre["t_cam"][act], axis=1)))
    return mism == 0, mism


def test_host_blas_matches_engine_fma_order():
    arrs = fg.cloud_arrays("C3_pi4")
    pos = arrs["positions"].astype(np.float64)
    for phi in (np.pi / 4, 0.7, 2.2):
        ok, mism = blas_order_matches(pos, phi)
        assert ok, (f"numpy/BLAS on this host rounds positions @ W.T differently from the engine's "
                    f"fma order in {mism} rows at phi={phi}: reference depth ties would order differently "
                    f"here (golden host: {fg.load()['host']})")


def test_golden_records_its_host():
    host = str(fg.load()["host"])
    assert "numpy" in host and len(host) > 10
