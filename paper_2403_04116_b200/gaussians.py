"""Learnable scene: radiative 3D Gaussians resident in HBM.

Restates the reference's data model (``pkg/src/xsplat/gaussians.py``):

* ``GaussianCloud.FIELDS`` = positions (N,3) mm, rotations (N,4) quaternions
  (w,x,y,z), log_scales (N,3) (log of per-axis std-dev, mm), raw_opacities (N,)
  (logit of opacity), features (N,N_f) radiation features
  (``gaussians.py:154-193``);
* ``basis_weights`` (N_f,) is fixed at construction, defaults to ones and is
  not learnable (``gaussians.py:188-193``);
* intensity i = sigmoid(F . lambda) is view-independent (``rirf``,
  ``gaussians.py:110-124``), opacity = sigmoid(raw) (``:222-224``), scale =
  exp(log_scale) (``:226-228``).

B200 layout: every learnable field is a view into ONE contiguous float32
device buffer ``[positions | rotations | log_scales | raw_opacities |
features]`` (27 floats per Gaussian at N_f = 16).  Gradients and both Adam
moments use the same layout, so the fused Adam kernel and the data-parallel
gradient all-reduce each see a single flat array.

Staleness (``StaleSplatsError``) is detected through torch's per-tensor
version counters instead of the reference's O(N) content sums
(``gaussians.py:259-270``): any in-place write to a field bumps its counter.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import InvalidParameterError

COV3_REGULARIZATION = 1e-9
COV2_LOWPASS = 0.3

PARAM_FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")


def default_device() -> torch.device:
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def field_widths(n_features: int) -> dict[str, int]:
    return {"positions": 3, "rotations": 4, "log_scales": 3, "raw_opacities": 1, "features": n_features}


def field_offsets(n: int, n_features: int) -> dict[str, tuple[int, int]]:
    """(start, stop) element offsets of every field inside the flat buffer."""
    out = {}
    pos = 0
    for f, wdt in field_widths(n_features).items():
        out[f] = (pos, pos + n * wdt)
        pos += n * wdt
    return out


def flat_size(n: int, n_features: int) -> int:
    return n * (11 + n_features)


def flat_views(flat: torch.Tensor, n: int, n_features: int) -> dict[str, torch.Tensor]:
    views = {}
    for f, (a, b) in field_offsets(n, n_features).items():
        v = flat[a:b]
        views[f] = v if f == "raw_opacities" else v.view(n, -1)
    return views


def sigmoid(x):
    """Numerically stable logistic on numpy input (two-branch form of
    ``gaussians.py:29-38``); host-side helper for tests and init."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return float(out) if out.ndim == 0 else out


def logit(p: float) -> float:
    if not 0.0 < p < 1.0:
        raise InvalidParameterError(f"logit argument must be in (0, 1), got {p}")
    return float(np.log(p) - np.log1p(-p))


def quaternions_to_rotations(q) -> np.ndarray:
    """Host float64 R(q/|q|) for (N,4) or (4,) quaternions (w,x,y,z)
    (``gaussians.py:47-69``).  The device kernels carry their own copy."""
    q = np.asarray(q, dtype=np.float64)
    single = q.ndim == 1
    q = np.atleast_2d(q)
    norm = np.sqrt(np.sum(q * q, axis=1, keepdims=True))
    if np.any(norm == 0):
        raise InvalidParameterError("zero quaternion")
    w, x, y, z = (q / norm).T
    r = np.stack(
        [
            1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
            2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
            2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y),
        ],
        axis=1,
    ).reshape(-1, 3, 3)
    return r[0] if single else r


@dataclass
class RadiativeGaussian:
    """One primitive, host-side (``gaussians.py:72-100``)."""

    position: np.ndarray
    rotation: np.ndarray
    log_scale: np.ndarray
    raw_opacity: float
    feature: np.ndarray

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.log_scale = np.asarray(self.log_scale, dtype=np.float64).reshape(3)
        self.feature = np.asarray(self.feature, dtype=np.float64).reshape(-1)
        self.raw_opacity = float(self.raw_opacity)

    @property
    def opacity(self) -> float:
        return float(sigmoid(self.raw_opacity))

    @property
    def scale(self) -> np.ndarray:
        return np.exp(self.log_scale)


def _as_f32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=torch.float32)
    return torch.as_tensor(np.array(x, dtype=np.float64), dtype=torch.float32, device=device)


class GaussianCloud:
    """N radiative Gaussians stored SoA in one float32 device buffer."""

    FIELDS = PARAM_FIELDS

    def __init__(
        self,
        positions,
        rotations,
        log_scales,
        raw_opacities,
        features,
        basis_weights=None,
        device=None,
    ):
        device = torch.device(device) if device is not None else default_device()
        pos = _as_f32(positions, device)
        feat = _as_f32(features, device)
        n = int(pos.shape[0]) if pos.ndim >= 1 else 0
        if n < 1:
            raise InvalidParameterError("cloud must contain at least one Gaussian")
        if feat.ndim != 2:
            raise InvalidParameterError("features must be 2-dimensional (N, n_features)")
        nf = int(feat.shape[1])
        src = {
            "positions": pos,
            "rotations": _as_f32(rotations, device),
            "log_scales": _as_f32(log_scales, device),
            "raw_opacities": _as_f32(raw_opacities, device).reshape(-1),
            "features": feat,
        }
        for name, width in (("positions", 3), ("rotations", 4), ("log_scales", 3)):
            if tuple(src[name].shape) != (n, width):
                raise InvalidParameterError(
                    f"{name} must have shape ({n}, {width}), got {tuple(src[name].shape)}"
                )
        if tuple(src["raw_opacities"].shape) != (n,) or feat.shape[0] != n:
            raise InvalidParameterError("attribute row counts disagree")
        if basis_weights is None:
            bw = torch.ones(nf, dtype=torch.float32, device=device)
        else:
            bw = _as_f32(basis_weights, device).reshape(-1).clone()
        if bw.shape[0] != nf:
            raise InvalidParameterError("basis_weights length must equal feature length")
        self._n = n
        self._nf = nf
        self._device = device
        self._flat = torch.empty(flat_size(n, nf), dtype=torch.float32, device=device)
        self._views = flat_views(self._flat, n, nf)
        for f in PARAM_FIELDS:
            self._views[f].copy_(src[f])
        self._basis = bw.contiguous()

    # --- construction helpers -------------------------------------------------
    @classmethod
    def from_flat(cls, flat: torch.Tensor, n: int, n_features: int, basis_weights: torch.Tensor):
        """Adopt an existing flat buffer (no copy) - used by density control."""
        obj = cls.__new__(cls)
        obj._n, obj._nf, obj._device = int(n), int(n_features), flat.device
        if flat.numel() != flat_size(n, n_features) or flat.dtype != torch.float32:
            raise InvalidParameterError("flat buffer has the wrong size or dtype")
        obj._flat = flat.contiguous()
        obj._views = flat_views(obj._flat, obj._n, obj._nf)
        obj._basis = basis_weights
        return obj

    @classmethod
    def from_gaussians(cls, gaussians, basis_weights=None, device=None):
        if not gaussians:
            raise InvalidParameterError("cloud must contain at least one Gaussian")
        return cls(
            np.stack([g.position for g in gaussians]),
            np.stack([g.rotation for g in gaussians]),
            np.stack([g.log_scale for g in gaussians]),
            np.array([g.raw_opacity for g in gaussians]),
            np.stack([g.feature for g in gaussians]),
            basis_weights=basis_weights,
            device=device,
        )

    # --- fields ---------------------------------------------------------------
    def _get(self, f):
        return self._views[f]

    def _set(self, f, value):
        v = self._views[f]
        value = _as_f32(value, self._device)
        if tuple(value.shape) != tuple(v.shape):
            raise InvalidParameterError(f"{f} must keep shape {tuple(v.shape)}")
        v.copy_(value)

    positions = property(lambda s: s._get("positions"), lambda s, v: s._set("positions", v))
    rotations = property(lambda s: s._get("rotations"), lambda s, v: s._set("rotations", v))
    log_scales = property(lambda s: s._get("log_scales"), lambda s, v: s._set("log_scales", v))
    raw_opacities = property(
        lambda s: s._get("raw_opacities"), lambda s, v: s._set("raw_opacities", v)
    )
    features = property(lambda s: s._get("features"), lambda s, v: s._set("features", v))

    @property
    def flat(self) -> torch.Tensor:
        return self._flat

    @property
    def basis_weights(self) -> torch.Tensor:
        return self._basis

    @property
    def device(self) -> torch.device:
        return self._device

    @property
    def n_points(self) -> int:
        return self._n

    @property
    def n_features(self) -> int:
        return self._nf

    @property
    def opacities(self) -> torch.Tensor:
        return torch.sigmoid(self.raw_opacities.double()).float()

    @property
    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales.double()).float()

    def intensities(self) -> torch.Tensor:
        """i = sigmoid(F . lambda) from the device kernel, bit-identical to the
        per-splat intensities every render produces (``gaussians.py:230-232``)."""
        from . import _native

        return _native.intensities(self)

    def normalize_rotations(self) -> None:
        q = self.rotations
        q.div_(torch.linalg.vector_norm(q, dim=1, keepdim=True))

    def mark_mutated(self) -> None:
        """Record an in-place write done by a CUDA kernel through a raw
        pointer (Adam), which torch's version counter cannot see."""
        torch.autograd.graph.increment_version(self._flat)

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i: int) -> RadiativeGaussian:
        return RadiativeGaussian(
            self.positions[i].cpu().numpy(),
            self.rotations[i].cpu().numpy(),
            self.log_scales[i].cpu().numpy(),
            float(self.raw_opacities[i]),
            self.features[i].cpu().numpy(),
        )

    def copy(self) -> "GaussianCloud":
        return GaussianCloud.from_flat(self._flat.clone(), self._n, self._nf, self._basis.clone())

    def to_numpy(self) -> dict[str, np.ndarray]:
        """float64 host copies of every field plus the basis weights."""
        out = {f: self._views[f].detach().cpu().double().numpy() for f in PARAM_FIELDS}
        out["basis_weights"] = self._basis.detach().cpu().double().numpy()
        return out

    def fingerprint(self) -> tuple:
        """Version token: changes whenever any field is written in place."""
        return (
            self._n,
            self._nf,
            self._flat.data_ptr(),
            self._flat._version,
            tuple(self._views[f]._version for f in PARAM_FIELDS),
        )


def covariance_3d(g: RadiativeGaussian) -> np.ndarray:
    r = quaternions_to_rotations(g.rotation)
    m = r * np.exp(g.log_scale)[None, :]
    return m @ m.T


def covariance_2d(cov3, jac, view_rot) -> np.ndarray:
    u = (np.asarray(jac) @ np.asarray(view_rot))[:2, :]
    return u @ np.asarray(cov3) @ u.T + COV2_LOWPASS * np.eye(2)


def rirf(feature, basis_weights):
    """Host float64 radiation intensity (``gaussians.py:110-124``)."""
    feature = np.asarray(feature, dtype=np.float64)
    basis_weights = np.asarray(basis_weights, dtype=np.float64)
    if feature.shape[-1] != basis_weights.shape[0]:
        raise InvalidParameterError(
            f"feature length {feature.shape[-1]} != weights length {basis_weights.shape[0]}"
        )
    if not (np.all(np.isfinite(feature)) and np.all(np.isfinite(basis_weights))):
        raise InvalidParameterError("feature and weights must be finite")
    return sigmoid(feature @ basis_weights)
