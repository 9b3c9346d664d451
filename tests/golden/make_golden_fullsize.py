"""Golden vectors from the REAL reference (xsplat 0.1.0) at BASELINE.json's
full sizes (C1 50,653 G at 256^2, C2 103,823 G at 512^2, C3
493,039 G at 512^2, C4 1,030,301 G at 1024^2).  Run in the build container (needs oracle/_ref,
built by oracle/build_ref.sh from /root/reference):

    python tests/golden/make_golden_fullsize.py     # -> tests/golden/fullsize.npz

Clouds come from the reference's own generator
(``acui.init_alternative("cuboid", CuboidSpec((100,)*3, (G,)*3, 2), 16, 0)``,
acui.py:132-155) rounded to float32, so the float64 reference and the
float32-parameter engine see identical inputs; the fixture stores a SHA-256
of those float32 arrays and the test checks the engine's generator
reproduces them before comparing anything.

Stored per case ``<case>/<key>``:

* ``cloud_sha`` - digest of the float32 cloud (positions, rotations,
  log_scales, raw_opacities, features in that order, C order);
* ``camera`` - (L_SO, L_SD, W, H, pitch, phi);
* ``active_sha``, ``entry_sha``, ``ranges_sha``, ``depths_sha`` - digests of
  the reference SplatList's active_indices (int64), entry_splat (int32,
  active-row form), tile_ranges (int64) and depths (float64 bits);
* ``tile_ranges`` and ``tile_sha`` (one 8-byte digest of each tile's
  entry_splat slice, so a mismatch points at its tiles);
* full arrays where small enough: C1 keeps entry_splat, radii, depths,
  image and (phi = 0.7) the kernel gradients and RenderGradients of
  dL/dI ~ N(0,1)/HW, seed 0 (SURVEY 8d's C1 unit of work); C2 at 0.7 the
  image, kernel gradients and the geometric RenderGradients fields for the
  same dL/dI; C3 at pi/4 and C4 at 0.7 the image (float32; the contract is
  1e-4 relative).

``host`` records the CPU model and numpy's BLAS that produced the float64
depths: the engine reproduces OpenBLAS dgemm's accumulation order
(``fma(w2, z, fma(w1, y, w0 * x))``), and tests/test_blas_guard.py fails
loudly if the numpy running the reference on a host departs from it.
"""

from __future__ import annotations

import hashlib
import io
import platform
import sys
import time
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from xsplat.acui import CuboidSpec, init_alternative  # noqa: E402
from xsplat.gaussians import GaussianCloud  # noqa: E402
from xsplat.geometry import ScannerConfig, extrinsic_from_angle, intrinsic_from_config  # noqa: E402
from xsplat.rasterizer import get_kernels, project_splats, render, render_backward, set_backend  # noqa: E402
from xsplat.trainer import PARAM_FIELDS  # noqa: E402

OUT = Path(__file__).resolve().parent / "fullsize.npz"
L_SO, L_SD = 1000.0, 1500.0
# (case, G, D, phi, what): "full" = render + backward, "image" = render, "bin" = project_splats only
CASES = (
    ("C1_0.7", 68, 256, 0.7, "full"),
    ("C1_pi4", 68, 256, np.pi / 4, "image"),
    ("C2_0.7", 88, 512, 0.7, "full"),
    ("C3_0", 152, 512, 0.0, "bin"),
    ("C3_pi4", 152, 512, np.pi / 4, "image"),
    ("C3_0.7", 152, 512, 0.7, "bin"),
    ("C4_0.7", 196, 1024, 0.7, "image"),
)
# RenderGradients fields stored for the larger "full" cases (the features
# gradient is g_int i (1 - i) lambda: pinned through k_g_int)
GRAD_FIELDS_LARGE = ("positions", "rotations", "log_scales", "raw_opacities", "screen_norms")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cloud_sha(fields: dict) -> str:
    h = hashlib.sha256()
    for f in PARAM_FIELDS:
        h.update(np.ascontiguousarray(np.asarray(fields[f], np.float32)).tobytes())
    return h.hexdigest()


def tile_digests(entry_splat: np.ndarray, ranges: np.ndarray) -> np.ndarray:
    out = np.zeros(ranges.shape[0], dtype=np.uint64)
    for t, (a, b) in enumerate(ranges):
        out[t] = np.frombuffer(hashlib.blake2b(entry_splat[a:b].tobytes(), digest_size=8).digest(), np.uint64)[0]
    return out


def f32_cloud(g: int):
    c = init_alternative("cuboid", CuboidSpec((100.0,) * 3, (g,) * 3, 2), 16, 0)
    f = {k: np.asarray(getattr(c, k), np.float32) for k in PARAM_FIELDS}
    cloud = GaussianCloud(*(f[k].astype(np.float64) for k in PARAM_FIELDS),
                          np.asarray(c.basis_weights, np.float64))
    return f, cloud


def host_info() -> str:
    model = platform.processor()
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    buf = io.StringIO()
    with redirect_stdout(buf):
        np.show_config()
    blas = [ln.strip() for ln in buf.getvalue().splitlines() if "openblas" in ln.lower() or "name:" in ln][:6]
    return f"{model} | numpy {np.__version__} | " + "; ".join(blas)


def main():
    set_backend("compiled")
    st: dict = {"host": np.array(host_info())}
    clouds: dict = {}
    for case, g, d, phi, what in CASES:
        t0 = time.perf_counter()
        if g not in clouds:
            clouds[g] = f32_cloud(g)
        fields, cloud = clouds[g]
        sc = ScannerConfig(L_SO, L_SD, d, d, 192.0 / d)
        ext, intr = extrinsic_from_angle(sc, phi), intrinsic_from_config(sc)
        p = case + "/"
        st[p + "cloud_sha"] = np.array(cloud_sha(fields))
        st[p + "n_points"] = np.array(cloud.n_points)
        st[p + "camera"] = np.array([L_SO, L_SD, d, d, 192.0 / d, phi])
        if what == "bin":
            sp = project_splats(cloud, ext, intr, (d, d))
        else:
            proj, sp = render(cloud, ext, intr, (d, d))
        st[p + "active_sha"] = np.array(sha(np.asarray(sp.active_indices, np.int64)))
        st[p + "entry_sha"] = np.array(sha(np.asarray(sp.entry_splat, np.int32)))
        st[p + "ranges_sha"] = np.array(sha(np.asarray(sp.tile_ranges, np.int64)))
        st[p + "depths_sha"] = np.array(sha(np.asarray(sp.depths, np.float64)))
        st[p + "n_entries"] = np.array(int(sp.entry_splat.size))
        st[p + "tile_ranges"] = np.asarray(sp.tile_ranges, np.int64)
        st[p + "tile_sha"] = tile_digests(np.asarray(sp.entry_splat, np.int32), np.asarray(sp.tile_ranges))
        if case.startswith("C1"):
            st[p + "entry_splat"] = np.asarray(sp.entry_splat, np.int32)
            st[p + "active_indices"] = np.asarray(sp.active_indices, np.int32)
            st[p + "radii"] = np.asarray(sp.radii, np.float64)
            st[p + "depths"] = np.asarray(sp.depths, np.float64)
        if what != "bin":
            st[p + "image"] = np.asarray(proj.pixels, np.float64 if case.startswith("C1") else np.float32)
        if what == "full":
            dl = np.random.default_rng(0).normal(size=(d, d)) / (d * d)
            gm, gc, gi, ga = get_kernels().backward_tiles(d, d, sp.means2d, sp.conics, sp.intensities,
                                                          sp.opacities, sp.entry_splat, sp.tile_ranges, dl)
            for k, v in (("k_g_mean", gm), ("k_g_conic", gc), ("k_g_int", gi), ("k_g_alpha", ga)):
                st[p + k] = np.asarray(v, np.float32)
            grads = render_backward(cloud, sp, dl)
            gfields = PARAM_FIELDS + ("screen_norms",) if case.startswith("C1") else GRAD_FIELDS_LARGE
            for f in gfields:
                st[p + "grad_" + f] = np.asarray(getattr(grads, f), np.float32)
            st[p + "grad_visible"] = np.asarray(grads.visible)
        print(f"{case}: N={cloud.n_points} E={sp.entry_splat.size} ({time.perf_counter() - t0:.1f} s)", flush=True)
    np.savez_compressed(OUT, **st)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
