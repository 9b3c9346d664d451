"""Voxel phantoms and the GPU cone-beam projector (training-target generator).

Mirrors ``pkg/src/xsplat/phantom.py``: additive axis-aligned primitives
(``Ellipsoid``, ``Cuboid``; ``phantom.py:39-113``) rasterised at voxel
centres into a ``VoxelPhantom`` centred on the origin (``:117-170``), the
default structured test object (``:173-187``), and ``project_phantom`` /
``project_all`` (``:190-250``): one ray per detector pixel through the
volume, trilinear samples at the midpoints of equal sub-steps, summed.

The primitives and the voxelisation are host numpy (they run once per
dataset); the projection is the ``xg_project_volume`` kernel
(csrc/xg_project.cu) - float64, sample positions bit-identical to the
reference's - which turns the reference's minutes of ``map_coordinates``
per 100-view 512^2 set into milliseconds.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import InvalidParameterError
from .geometry import ScannerConfig, viewing_rotation

DEFAULT_STEP_FACTOR = 0.25  # ray-march step / smallest voxel edge (phantom.py:20-22)
DEFAULT_NOISE_LEVEL = 0.03


def _vec3(x, what: str) -> np.ndarray:
    a = np.asarray(x, dtype=np.float64)
    if a.shape != (3,):
        raise InvalidParameterError(f"{what}: center and size must be 3-vectors")
    return a


def _validated(center, size, density, what: str):
    c, s = _vec3(center, what), _vec3(size, what)
    if (s <= 0).any():
        raise InvalidParameterError(f"{what}: size must be positive, got {s}")
    if density < 0:
        raise InvalidParameterError(f"{what}: density must be >= 0, got {density}")
    return c, s, float(density)


@dataclass
class Ellipsoid:
    """Axis-aligned ellipsoid adding ``density`` inside its surface."""

    center: np.ndarray
    semi_axes: np.ndarray
    density: float

    def __post_init__(self):
        self.center, self.semi_axes, self.density = _validated(self.center, self.semi_axes, self.density,
                                                               "ellipsoid")

    def bounds(self):
        return self.center - self.semi_axes, self.center + self.semi_axes

    def evaluate(self, x, y, z):
        q = sum(((c - o) / a) ** 2 for c, o, a in zip((x, y, z), self.center, self.semi_axes))
        return np.where(q <= 1.0, self.density, 0.0)

    def to_dict(self) -> dict:
        return {"kind": "ellipsoid", "center": self.center.tolist(), "semi_axes": self.semi_axes.tolist(),
                "density": self.density}


@dataclass
class Cuboid:
    """Axis-aligned box adding ``density`` inside."""

    center: np.ndarray
    half_extents: np.ndarray
    density: float

    def __post_init__(self):
        self.center, self.half_extents, self.density = _validated(self.center, self.half_extents,
                                                                  self.density, "cuboid")

    def bounds(self):
        return self.center - self.half_extents, self.center + self.half_extents

    def evaluate(self, x, y, z):
        inside = np.ones(np.shape(x), dtype=bool)
        for c, o, e in zip((x, y, z), self.center, self.half_extents):
            inside &= np.abs(c - o) <= e
        return np.where(inside, self.density, 0.0)

    def to_dict(self) -> dict:
        return {"kind": "cuboid", "center": self.center.tolist(), "half_extents": self.half_extents.tolist(),
                "density": self.density}


_KINDS = {"ellipsoid": (Ellipsoid, "semi_axes"), "cuboid": (Cuboid, "half_extents")}


def primitive_from_dict(d: dict):
    kind = d.get("kind")
    if kind not in _KINDS:
        raise InvalidParameterError(f"unknown primitive kind {kind!r}")
    cls, size_key = _KINDS[kind]
    return cls(d["center"], d[size_key], d["density"])


@dataclass
class VoxelPhantom:
    """Non-negative density volume on a regular grid centred on the origin."""

    densities: np.ndarray
    voxel_size: np.ndarray
    primitives: list = field(default_factory=list)

    def __post_init__(self):
        self.densities = np.ascontiguousarray(self.densities, dtype=np.float64)
        self.voxel_size = np.asarray(self.voxel_size, dtype=np.float64)
        if self.densities.ndim != 3:
            raise InvalidParameterError("densities must be a 3-D array")
        if self.voxel_size.shape != (3,) or (self.voxel_size <= 0).any():
            raise InvalidParameterError("voxel_size must be three positive reals")
        if not np.isfinite(self.densities).all() or (self.densities < 0).any():
            raise InvalidParameterError("densities must be finite and >= 0")
        self._device = None

    @property
    def grid(self) -> tuple[int, int, int]:
        return tuple(int(m) for m in self.densities.shape)

    @property
    def extent(self) -> np.ndarray:
        return np.array(self.grid) * self.voxel_size

    def device_volume(self, device="cuda") -> torch.Tensor:
        """The densities resident on the GPU (uploaded once, 8 B/voxel)."""
        if self._device is None or str(self._device.device) != str(torch.device(device)):
            self._device = torch.as_tensor(self.densities, device=device)
        return self._device


def make_phantom(primitives, grid, voxel_size) -> VoxelPhantom:
    """Sum the primitives at voxel centres (phantom.py:143-170)."""
    grid = tuple(int(m) for m in grid)
    vs = np.broadcast_to(np.asarray(voxel_size, dtype=np.float64), (3,)).copy()
    if min(grid) < 1 or (vs <= 0).any():
        raise InvalidParameterError("grid must be >= 1 and voxel_size positive")
    extent = np.array(grid) * vs
    centres = [(np.arange(m) + 0.5) * s - e / 2.0 for m, s, e in zip(grid, vs, extent)]
    x, y, z = np.meshgrid(*centres, indexing="ij")
    dens = np.zeros(grid)
    for prim in primitives:
        lo, hi = prim.bounds()
        if (lo < -extent / 2.0 - 1e-9).any() or (hi > extent / 2.0 + 1e-9).any():
            raise InvalidParameterError(f"primitive {prim.to_dict()['kind']} extends outside the volume")
        dens += prim.evaluate(x, y, z)
    return VoxelPhantom(dens, vs, list(primitives))


def default_phantom_primitives(extent) -> list:
    """The structured test object of phantom.py:173-187: a soft body with
    embedded blobs and boxes, laid out in fractions of the extent."""
    s = np.asarray(extent, dtype=np.float64)
    ell = [((0.0, 0.0, 0.0), (0.40, 0.40, 0.40), 0.35),
           ((0.10, -0.06, 0.05), (0.16, 0.20, 0.14), 0.45),
           ((-0.15, 0.12, -0.08), (0.10, 0.08, 0.12), 0.60),
           ((0.18, 0.15, -0.12), (0.05, 0.05, 0.05), 1.00),
           ((-0.05, 0.02, -0.18), (0.035, 0.035, 0.035), 1.20)]
    box = [((-0.12, -0.16, 0.10), (0.08, 0.06, 0.10), 0.55),
           ((0.02, 0.18, 0.14), (0.05, 0.09, 0.04), 0.80)]
    return ([Ellipsoid(np.array(c) * s, np.array(a) * s, d) for c, a, d in ell]
            + [Cuboid(np.array(c) * s, np.array(a) * s, d) for c, a, d in box])


def cone_view(scanner: ScannerConfig, phi: float) -> nat.XgConeView:
    """Source position and rotation of one view, computed on the host with
    the reference's own functions (math.sin / math.cos, viewing_rotation)."""
    v = nat.XgConeView()
    d = scanner.source_object_distance
    v.source[:] = (d * np.cos(phi), d * np.sin(phi), 0.0)
    v.rot[:] = np.asarray(viewing_rotation(phi), dtype=np.float64).reshape(-1).tolist()
    v.focal = float(scanner.focal_pixels)
    v.width, v.height = int(scanner.detector_width), int(scanner.detector_height)
    return v


class Projector:
    """Workspace + launch state of ``xg_project_volume`` for one phantom and
    one detector size."""

    def __init__(self, ph: VoxelPhantom, scanner: ScannerConfig, device="cuda"):
        self.ph, self.scanner = ph, scanner
        self.dens = ph.device_volume(device)
        h, w = scanner.detector_height, scanner.detector_width
        self.ws = torch.empty(int(nat.lib().xg_project_workspace_bytes(h, w)), dtype=torch.uint8, device=device)
        self.vol = nat.XgVolume()
        self.vol.densities = self.dens.data_ptr()
        self.vol.m[:] = list(ph.grid)
        self.vol.voxel_size[:] = ph.voxel_size.tolist()

    def project(self, phi: float, out: torch.Tensor, step_factor: float = DEFAULT_STEP_FACTOR) -> torch.Tensor:
        if not 0 < step_factor <= 0.5:
            raise InvalidParameterError("step_factor must be in (0, 0.5]")
        if not math.isfinite(phi):
            raise InvalidParameterError(f"angle must be finite, got {phi}")
        view = cone_view(self.scanner, phi)
        nat.check(nat.lib().xg_project_volume(ctypes.byref(self.vol), ctypes.byref(view), float(step_factor),
                                              nat.ptr(out, "out"), self.ws.data_ptr(), self.ws.numel(),
                                              nat.stream()), "xg_project_volume")
        return out


def project_phantom(ph: VoxelPhantom, scanner: ScannerConfig, phi: float,
                    step_factor: float = DEFAULT_STEP_FACTOR) -> torch.Tensor:
    """Raw line integrals (H, W) float64 of one view, on the GPU."""
    out = torch.empty((scanner.detector_height, scanner.detector_width), dtype=torch.float64, device="cuda")
    return Projector(ph, scanner, out.device).project(phi, out, step_factor)


def project_all(ph: VoxelPhantom, scanner: ScannerConfig, step_factor: float = DEFAULT_STEP_FACTOR) -> torch.Tensor:
    """Raw projections (n, H, W) float64 for every configured angle, on the GPU."""
    angles = np.asarray(scanner.angles, dtype=np.float64)
    out = torch.empty((angles.size, scanner.detector_height, scanner.detector_width), dtype=torch.float64,
                      device="cuda")
    pr = Projector(ph, scanner, out.device)
    for i, phi in enumerate(angles):
        pr.project(float(phi), out[i], step_factor)
    return out
