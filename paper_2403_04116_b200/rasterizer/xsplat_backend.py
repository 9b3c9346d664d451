"""The reference-side binding: a ``"cuda"`` kernel backend for xsplat itself.

xsplat picks its blend kernels from a registry (``rasterizer/backend.py:
20-46``: ``_BACKENDS``, ``set_backend``, ``get_kernels``); each backend is a
module exporting ``forward_tiles`` / ``backward_tiles`` over float64 numpy
arrays in the active-row layout (``_kernels.pyx:23-32, 77-87``).  This module
is exactly that contract - numpy in, numpy out - served by
``xg_forward_tiles_f64`` / ``xg_backward_tiles_f64`` of libxgauss.so
(through :mod:`.tiles`): the reference's float64 arithmetic in its
operation order, so xsplat's own tests and its backend lockstep tolerance
(1e-12) hold on it; ``register`` adds it to an imported xsplat as
``_BACKENDS["cuda"]``.  It is the stub INTEGRATION.md section 2 shows, made
a tested module: tests/test_gpu_xsplat_plugin.py runs xsplat's own rasterizer
and gradient suites with it.

Host arrays are copied to the device per call and results copied back, as
the reference's callers expect fresh numpy arrays (``frontend.py:223-232``,
``backward.py:49-59``).  (The engine's own render path composites in
float32 with the north_star tolerance of 1e-4; ``tiles.forward_tiles`` /
``backward_tiles`` serve that path through the same contract.)
"""

from __future__ import annotations

import numpy as np

from . import tiles


def forward_tiles(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges) -> np.ndarray:
    """_kernels.pyx:23-74 contract: float64 [h, w] image."""
    return tiles.forward_tiles_f64(h, w, means2d, conics, intensities, opacities, entry_splat,
                                   tile_ranges).cpu().numpy()


def backward_tiles(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges, dl_dimage):
    """_kernels.pyx:77-178 contract: (g_mean [A,2], g_conic [A,3], g_int [A], g_alpha [A]) float64."""
    out = tiles.backward_tiles_f64(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                                   dl_dimage)
    return tuple(t.cpu().numpy() for t in out)


def register(backend_module, name: str = "cuda") -> None:
    """Add this module to an imported ``xsplat.rasterizer.backend`` registry
    (the maintainer's one-line change: ``_BACKENDS["cuda"] = _cuda_backend``)."""
    import sys

    backend_module._BACKENDS[name] = sys.modules[__name__]
