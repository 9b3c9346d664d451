"""Forward rasterization API: project, bin, composite - on the GPU.

Mirrors ``xsplat.rasterizer.frontend`` (``pkg/src/xsplat/rasterizer/
frontend.py``) call for call:

* ``project_splats(cloud, ext, intr, image_shape) -> SplatList`` (:104-194)
* ``render(cloud, ext, intr, image_shape) -> (Projection, SplatList)`` (:208-233)
* ``render_view(cloud, scanner, phi)`` (:236-242)
* ``blend_pixel`` (:245-256) and ``brute_force_render`` (:259-289), the
  reference's own test oracles

Results are CUDA tensors (float32 images; the per-splat geometry the
reference exposes is float64 because the projection runs in float64).
``SplatList`` keeps the per-Gaussian device buffers of the view and exposes
the reference's active-row fields (``active_indices``, ``means2d``,
``entry_splat`` as active-row indices, ...) as lazily compacted views.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import _native as nat
from ..engine import Frame, tile_grid
from ..errors import InvalidParameterError
from ..gaussians import GaussianCloud
from ..geometry import (
    ExtrinsicMatrix,
    IntrinsicMatrix,
    ScannerConfig,
    camera_pod,
    extrinsic_from_angle,
    intrinsic_from_config,
)
from .constants import POWER_CUTOFF, SIGMA_CLAMP, TRANSMITTANCE_FLOOR


@dataclass
class Projection:
    """A rendered detector image (CUDA float32 [H, W]) and its azimuth."""

    pixels: torch.Tensor
    angle: float


@dataclass
class RenderGradients:
    """Cloud-shaped gradients (views into one flat float32 buffer laid out
    like ``GaussianCloud.flat``), plus ``screen_norms`` and ``visible``
    (frontend.py:81-97)."""

    positions: torch.Tensor
    rotations: torch.Tensor
    log_scales: torch.Tensor
    raw_opacities: torch.Tensor
    features: torch.Tensor
    screen_norms: torch.Tensor
    visible: torch.Tensor
    flat: torch.Tensor | None = None


class SplatList:
    """Screen-space state of one view (frontend.py:47-78)."""

    def __init__(self, frame: Frame, cloud: GaussianCloud, ext: ExtrinsicMatrix, intr: IntrinsicMatrix,
                 image_shape, n_active: int, n_entries: int):
        self._frame = frame
        self.image_shape = (int(image_shape[0]), int(image_shape[1]))
        self.view_rotation = np.array(ext.rotation, dtype=np.float64)
        self.focal = intr.focal
        self.angle = ext.angle
        self.n_total = cloud.n_points
        self.cloud_fingerprint = cloud.fingerprint()
        self._n_active = int(n_active)
        self._n_entries = int(n_entries)
        self._active_idx = None
        self._rowmap = None

    # --- engine-side views ----------------------------------------------------
    @property
    def frame(self) -> Frame:
        return self._frame

    @property
    def n_active(self) -> int:
        return self._n_active

    @property
    def n_entries(self) -> int:
        return self._n_entries

    @property
    def order(self) -> torch.Tensor:
        """Cloud rows in (depth, index) order; the first ``n_active`` are active."""
        return self._frame.order[: self._n_active]

    @property
    def entry_ids(self) -> torch.Tensor:
        """Per-entry cloud row (the engine's native entry payload)."""
        return self._frame.entry_splat[: self._n_entries]

    @property
    def tiles_touched(self) -> torch.Tensor:
        return self._frame.tiles_touched

    @property
    def tile_rects(self) -> torch.Tensor:
        """[A, 4] (tx0, ty0, tx1, ty1) of the active rows."""
        return self._frame.rect[self.active_indices].to(torch.int64) & 0xFFFF

    # --- reference fields -----------------------------------------------------
    @property
    def active_indices(self) -> torch.Tensor:
        if self._active_idx is None:
            self._active_idx = torch.nonzero(self._frame.tiles_touched > 0).reshape(-1)
        return self._active_idx

    def _rows(self, t: torch.Tensor) -> torch.Tensor:
        return t[self.active_indices]

    def _extra(self, name):
        if self._frame.extras is None:
            raise InvalidParameterError(f"{name} was not recorded for this SplatList (engine-internal frame)")
        return self._rows(self._frame.extras[name])

    @property
    def means2d(self) -> torch.Tensor:
        return self._rows(self._frame.mean2d)

    @property
    def cov2d(self) -> torch.Tensor:
        return self._extra("cov2d")

    @property
    def conics(self) -> torch.Tensor:
        return self._extra("conic")

    @property
    def depths(self) -> torch.Tensor:
        return self._extra("depth")

    @property
    def t_cam(self) -> torch.Tensor:
        return self._extra("t_cam")

    @property
    def radii(self) -> torch.Tensor:
        return self._extra("radius")

    @property
    def opacities(self) -> torch.Tensor:
        return self._extra("opacity")

    @property
    def intensities(self) -> torch.Tensor:
        return self._rows(self._frame.inten)

    @property
    def entry_splat(self) -> torch.Tensor:
        """Active-row index per entry (int32), as the reference stores it."""
        if self._rowmap is None:
            act = (self._frame.tiles_touched > 0).to(torch.int32)
            self._rowmap = (torch.cumsum(act, 0) - 1).to(torch.int32)
        return self._rowmap[self.entry_ids.to(torch.int64)]

    @property
    def tile_ranges(self) -> torch.Tensor:
        return self._frame.tile_ranges


def _check_cloud(cloud: GaussianCloud) -> None:
    if cloud.n_points < 1:
        raise InvalidParameterError("cloud must contain at least one Gaussian")
    nat.require_cuda(cloud.flat, "cloud")


def _prepare(cloud, ext, intr, image_shape, extras: bool, composite: bool = False) -> tuple[Frame, SplatList]:
    """Preprocess + bin one view (one host sync: the entry count).  With
    ``composite`` the tracking forward is queued BEFORE that sync (it skips
    itself on the device if the entry buffer overflowed, and runs again on
    the re-binned lists), so the GPU never idles at the read."""
    _check_cloud(cloud)
    h, w = (int(v) for v in image_shape)
    if h < 1 or w < 1:
        raise InvalidParameterError(f"image shape must be positive, got {(h, w)}")
    frame = Frame(cloud.n_points, h, w, cloud.device, entry_capacity=_capacity_hint(cloud, h, w),
                  extras=extras)
    frame.preprocess(cloud, camera_pod(ext, intr, (h, w)))
    if composite:
        frame.bin_async()
        frame.composite()
        if frame.finish_bin():
            frame.composite()
        c = frame.last_counters
        active, entries, status = int(c[nat.XG_CTR_ACTIVE]), int(c[nat.XG_CTR_ENTRIES]), int(c[nat.XG_CTR_STATUS])
        nat.raise_for_status(status & ~nat.XG_ST_ENTRY_OVERFLOW)
    else:
        active, entries, _ = frame.ensure_binned()
    _remember_capacity(cloud, h, w, entries)
    return frame, SplatList(frame, cloud, ext, intr, (h, w), active, entries)


_CAP_HINTS: dict = {}


def _capacity_hint(cloud, h, w) -> int:
    return _CAP_HINTS.get((cloud.n_points, h, w), max(16 * cloud.n_points, 4096))


def _remember_capacity(cloud, h, w, entries) -> None:
    key = (cloud.n_points, h, w)
    _CAP_HINTS[key] = max(_CAP_HINTS.get(key, 0), int(entries * 1.25) + 4096)


def project_splats(cloud: GaussianCloud, ext: ExtrinsicMatrix, intr: IntrinsicMatrix,
                   image_shape) -> SplatList:
    """Projection, culling, tile rects, binning (frontend.py:104-194)."""
    _, splats = _prepare(cloud, ext, intr, image_shape, extras=True)
    return splats


def render(cloud: GaussianCloud, ext: ExtrinsicMatrix, intr: IntrinsicMatrix,
           image_shape) -> tuple[Projection, SplatList]:
    """Rasterize the cloud into a detector image (frontend.py:208-233)."""
    frame, splats = _prepare(cloud, ext, intr, image_shape, extras=True, composite=True)
    return Projection(frame.image, splats.angle), splats


def render_view(cloud: GaussianCloud, scanner: ScannerConfig, phi: float) -> tuple[Projection, SplatList]:
    ext = extrinsic_from_angle(scanner, phi)
    intr = intrinsic_from_config(scanner)
    return render(cloud, ext, intr, (scanner.detector_height, scanner.detector_width))


def blend_pixel(ordered) -> float:
    """Scalar front-to-back composite of (intensity, sigma) pairs - the
    closed-form check of Eq. 10 (frontend.py:245-256); host-side."""
    acc = 0.0
    trans = 1.0
    for intensity, sigma in ordered:
        if not 0.0 <= sigma < 1.0:
            raise InvalidParameterError(f"sigma must be in [0, 1), got {sigma}")
        if trans < TRANSMITTANCE_FLOOR:
            break
        acc += intensity * sigma * trans
        trans *= 1.0 - sigma
    return acc


def brute_force_render(cloud: GaussianCloud, ext: ExtrinsicMatrix, intr: IntrinsicMatrix,
                       image_shape) -> Projection:
    """Untiled oracle (frontend.py:259-289): every active splat against every
    pixel in one global (depth, index) order, same cut-offs.  Implemented by
    handing the compositing kernel, for every tile, the full global list
    instead of the tile's binned list.  Quadratic - test-sized scenes only."""
    frame, splats = _prepare(cloud, ext, intr, image_shape, extras=False)
    a = splats.n_active
    h, w = splats.image_shape
    if a == 0:
        return Projection(torch.zeros((h, w), dtype=torch.float32, device=cloud.device), splats.angle)
    t = frame.n_tiles
    glob = frame.order[:a].clone()
    frame.set_capacity(a * t)
    frame.entry_splat[: a * t] = glob.repeat(t)
    starts = torch.arange(t, dtype=torch.int64, device=cloud.device) * a
    frame.tile_ranges[:, 0] = starts
    frame.tile_ranges[:, 1] = starts + a
    frame.composite()
    return Projection(frame.image, splats.angle)


__all__ = [
    "POWER_CUTOFF",
    "SIGMA_CLAMP",
    "TRANSMITTANCE_FLOOR",
    "Projection",
    "RenderGradients",
    "SplatList",
    "blend_pixel",
    "brute_force_render",
    "project_splats",
    "render",
    "render_view",
    "tile_grid",
]

