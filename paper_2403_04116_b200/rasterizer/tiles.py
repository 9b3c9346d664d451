"""The reference's kernel-backend contract, served by the CUDA library.

``xsplat`` selects blend kernels through a registry (``rasterizer/
backend.py:20-46``); each backend exports ``forward_tiles`` and
``backward_tiles`` over active-row arrays (``_kernels.pyx:23-32, 77-87``).
Here there is one backend, ``"cuda"`` - no dispatch, no CPU fallback - and
its two functions call ``xg_forward_tiles`` / ``xg_backward_tiles`` of
libxgauss.so.  Inputs may be numpy arrays or tensors; they are moved to the
current CUDA device, results are CUDA float64 tensors.
"""

from __future__ import annotations

import types

import torch

from .. import _native as nat

_BACKEND = "cuda"


def available_backends() -> tuple[str, ...]:
    return (_BACKEND,)


def active_backend() -> str:
    return _BACKEND


def set_backend(name: str) -> None:
    if name != _BACKEND:
        raise ValueError(f"unknown backend {name!r}; available: {available_backends()}")


def _dev(x, dtype) -> torch.Tensor:
    t = torch.as_tensor(x)
    return t.to(device="cuda", dtype=dtype).contiguous()


def _common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges, workspace: bool = True):
    m = _dev(means2d, torch.float64).reshape(-1, 2)
    c = _dev(conics, torch.float64).reshape(-1, 3)
    i = _dev(intensities, torch.float64).reshape(-1)
    o = _dev(opacities, torch.float64).reshape(-1)
    e = _dev(entry_splat, torch.int32).reshape(-1)
    r = _dev(tile_ranges, torch.int64).reshape(-1, 2)
    n = m.shape[0]
    if not workspace:
        return m, c, i, o, e, r, n, None
    ws = torch.empty(int(nat.lib().xg_tiles_workspace_bytes(n, int(h), int(w))), dtype=torch.uint8,
                     device="cuda")
    return m, c, i, o, e, r, n, ws


def forward_tiles(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges) -> torch.Tensor:
    m, c, i, o, e, r, n, ws = _common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges)
    img = torch.zeros((int(h), int(w)), dtype=torch.float64, device="cuda")
    nat.check(
        nat.lib().xg_forward_tiles(int(h), int(w), m.data_ptr(), c.data_ptr(), i.data_ptr(), o.data_ptr(),
                                   e.data_ptr(), e.numel(), r.data_ptr(), n, img.data_ptr(), ws.data_ptr(),
                                   ws.numel(), nat.stream()),
        "xg_forward_tiles",
    )
    return img


def backward_tiles(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges, dl_dimage):
    m, c, i, o, e, r, n, ws = _common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges)
    dl = _dev(dl_dimage, torch.float64).reshape(int(h), int(w))
    g_mean = torch.zeros((n, 2), dtype=torch.float64, device="cuda")
    g_conic = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    g_int = torch.zeros(n, dtype=torch.float64, device="cuda")
    g_alpha = torch.zeros(n, dtype=torch.float64, device="cuda")
    nat.check(
        nat.lib().xg_backward_tiles(int(h), int(w), m.data_ptr(), c.data_ptr(), i.data_ptr(), o.data_ptr(),
                                    e.data_ptr(), e.numel(), r.data_ptr(), n, dl.data_ptr(), g_mean.data_ptr(),
                                    g_conic.data_ptr(), g_int.data_ptr(), g_alpha.data_ptr(), ws.data_ptr(),
                                    ws.numel(), nat.stream()),
        "xg_backward_tiles",
    )
    return g_mean, g_conic, g_int, g_alpha


def forward_tiles_f64(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges) -> torch.Tensor:
    """forward_tiles at the reference's precision (xg_forward_tiles_f64:
    float64 in _kernels.pyx's operation order)."""
    m, c, i, o, e, r, n, _ = _common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                                     workspace=False)
    img = torch.empty((int(h), int(w)), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().xg_forward_tiles_f64(int(h), int(w), m.data_ptr(), c.data_ptr(), i.data_ptr(),
                                             o.data_ptr(), e.data_ptr(), e.numel(), r.data_ptr(), n,
                                             img.data_ptr(), nat.stream()), "xg_forward_tiles_f64")
    return img


def backward_tiles_f64(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges, dl_dimage):
    """backward_tiles at the reference's precision (xg_backward_tiles_f64)."""
    m, c, i, o, e, r, n, _ = _common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                                     workspace=False)
    dl = _dev(dl_dimage, torch.float64).reshape(int(h), int(w))
    g_mean = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    g_conic = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    g_int = torch.empty(n, dtype=torch.float64, device="cuda")
    g_alpha = torch.empty(n, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().xg_backward_tiles_f64(int(h), int(w), m.data_ptr(), c.data_ptr(), i.data_ptr(),
                                              o.data_ptr(), e.data_ptr(), e.numel(), r.data_ptr(), n,
                                              dl.data_ptr(), g_mean.data_ptr(), g_conic.data_ptr(),
                                              g_int.data_ptr(), g_alpha.data_ptr(), nat.stream()),
              "xg_backward_tiles_f64")
    return g_mean, g_conic, g_int, g_alpha


_KERNELS = types.SimpleNamespace(forward_tiles=forward_tiles, backward_tiles=backward_tiles)


def get_kernels():
    return _KERNELS

