"""ctypes binding of libxgauss.so (include/xgauss.h).

This is the drop-in boundary: the Python API of the package mirrors the
reference's (``xsplat``) and every compute step below it is one of the C-ABI
entry points declared in ``include/xgauss.h``.  There is no CPU fallback -
if the library is missing, or a tensor is not on a CUDA device, the call
fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import (
    InvalidParameterError,
    NativeError,
    NumericalDegeneracyError,
    TrainingDivergenceError,
)

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libxgauss.so"

XG_OK = 0
XG_ST_ZERO_QUAT = 0x1
XG_ST_DEGENERATE = 0x2
XG_ST_NONFINITE_FEAT = 0x4
XG_ST_ENTRY_OVERFLOW = 0x8
XG_ST_GRAD_SHIFT = 8
XG_ST_PEER_TIMEOUT = 0x10
XG_PEER_MAX = 8
XG_CTR_ACTIVE, XG_CTR_ENTRIES, XG_CTR_STATUS, XG_CTR_STICKY, XG_CTR_QUEUE = 0, 1, 2, 4, 5
XG_CTR_ITEMS = 6
XG_CTR_L1 = 8  # words 8-9: the fused-L1 double, zeroed by xg_preprocess_fwd
XG_NCOUNTERS = 10
XG_ABI_VERSION = 5
XG_REPLAY_CHUNK = 256
XG_MAX_BATCH = 16
PARAM_FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")

c_void_p = ctypes.c_void_p
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double
c_size = ctypes.c_size_t


class XgCloud(ctypes.Structure):
    _fields_ = [("params", c_void_p), ("basis", c_void_p), ("n", c_i64), ("n_features", c_i32), ("_pad", c_i32),
                ("intensities", c_void_p), ("invariants", c_void_p)]


class XgVolume(ctypes.Structure):
    _fields_ = [("densities", c_void_p), ("m", c_i32 * 3), ("_pad", c_i32), ("voxel_size", c_f64 * 3)]


class XgConeView(ctypes.Structure):
    _fields_ = [("source", c_f64 * 3), ("rot", c_f64 * 9), ("focal", c_f64), ("width", c_i32), ("height", c_i32)]


class XgPeerGroup(ctypes.Structure):
    """xg_peer_group (include/xgauss.h): every rank's peer-mapped buffers."""

    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("epoch", ctypes.c_uint32),
        ("grads", c_void_p * XG_PEER_MAX),
        ("xbuf", c_void_p * XG_PEER_MAX),
        ("sync", c_void_p * XG_PEER_MAX),
    ]


class XgSplats(ctypes.Structure):
    _fields_ = [
        ("mean2d", c_void_p),
        ("coef", c_void_p),
        ("inten", c_void_p),
        ("rect", c_void_p),
        ("n_tiles", c_void_p),
        ("depth_key", c_void_p),
        ("order", c_void_p),
        ("entry_splat", c_void_p),
        ("tile_ranges", c_void_p),
        ("counters", c_void_p),
        ("n", c_i64),
        ("entry_capacity", c_i64),
        ("tile_order", c_void_p),
        ("unit_cost", c_void_p),
        ("unit_order", c_void_p),
        ("replay_ckpt", c_void_p),
        ("replay_items", c_void_p),
        ("replay_slots", c_i64),
    ]


class XgSplatExtras(ctypes.Structure):
    _fields_ = [(f, c_void_p) for f in ("cov2d", "conic", "depth", "t_cam", "radius", "opacity")]


# name -> (restype, argtypes); every symbol include/xgauss.h declares.
SIGNATURES = {
    "xg_abi_version": (c_i32, []),
    "xg_last_error": (ctypes.c_char_p, []),
    "xg_kernel_launches": (ctypes.c_uint64, []),
    "xg_tiles_x": (c_i32, [c_void_p]),
    "xg_tiles_y": (c_i32, [c_void_p]),
    "xg_bin_workspace_bytes": (c_size, [c_i64, c_i64, c_i32]),
    "xg_replay_slots": (c_i64, [c_i64, c_i32]),
    "xg_preprocess_fwd": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "xg_bin_sort": (c_i32, [c_void_p, c_void_p, c_void_p, c_size, c_void_p]),
    "xg_composite_fwd": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "xg_composite_fwd_train": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p]),
    "xg_composite_train_pair": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_f32, c_void_p, c_void_p],
    ),
    "xg_composite_bwd": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_f32, c_void_p, c_void_p],
    ),
    "xg_entry_grad_bytes": (c_size, [c_i64, c_i64]),
    "xg_composite_bwd_entries": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_f32, c_void_p, c_size, c_void_p],
    ),
    "xg_reduce_entry_grads": (c_i32, [c_void_p, c_void_p, c_void_p, c_size, c_void_p, c_void_p]),
    "xg_preprocess_bwd": (c_i32, [c_void_p] * 15),
    "xg_check_finite": (c_i32, [c_void_p, c_i64, c_i32, c_void_p, c_void_p]),
    "xg_check_finite_range": (c_i32, [c_void_p, c_i64, c_i32, c_i64, c_i64, c_void_p, c_void_p]),
    "xg_adam": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_void_p, c_f64, c_f64, c_f64, c_f64, c_f64,
         c_void_p, c_void_p],
    ),
    "xg_adam_range": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_void_p, c_f64, c_f64, c_f64, c_f64, c_f64,
         c_void_p, c_i64, c_i64, c_void_p],
    ),
    "xg_adam_renorm": (c_i32, [c_void_p, c_i64, c_i32, c_void_p, c_void_p]),
    "xg_peer_slice": (c_i64, [c_i64, c_i32, c_i32]),
    "xg_peer_reduce_scatter": (c_i32, [c_void_p, c_i64, c_i32, c_void_p, c_void_p]),
    "xg_peer_allgather_adam": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_void_p, c_f64, c_f64, c_f64, c_f64, c_f64,
         c_void_p, c_void_p],
    ),
    "xg_densify_mark": (
        c_i32,
        [c_void_p, c_i64, c_i32, c_void_p, c_void_p, c_f64, c_f64, c_f64, c_void_p, c_void_p, c_void_p],
    ),
    "xg_densify_scratch_bytes": (c_size, [c_i64]),
    "xg_densify_apply": (
        c_i32,
        [c_void_p, c_void_p, c_void_p, c_i64, c_i32, c_void_p, c_void_p, c_void_p, c_f64, c_i32, c_void_p,
         c_void_p, c_void_p, c_i64, c_void_p, c_void_p],
    ),
    "xg_intensities": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "xg_view_invariants": (c_i32, [c_void_p, c_void_p, c_void_p]),
    "xg_tiles_workspace_bytes": (c_size, [c_i64, c_i32, c_i32]),
    "xg_ssim_workspace_bytes": (c_size, [c_i32, c_i32]),
    "xg_composite_batch_workspace_bytes": (c_size, [c_void_p, c_i32]),
    "xg_composite_fwd_batch": (c_i32, [c_void_p, c_void_p, c_void_p, c_i32, c_void_p, c_size, c_void_p]),
    "xg_project_workspace_bytes": (c_size, [c_i32, c_i32]),
    "xg_project_volume": (c_i32, [c_void_p, c_void_p, c_f64, c_void_p, c_void_p, c_size, c_void_p]),
    "xg_ssim": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, c_i32, c_f64, c_void_p, c_void_p, c_void_p, c_f64,
                        c_f64, c_void_p, c_size, c_void_p]),
    "xg_forward_tiles": (
        c_i32,
        [c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p,
         c_void_p, c_size, c_void_p],
    ),
    "xg_forward_tiles_f64": (
        c_i32, [c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p,
                c_void_p],
    ),
    "xg_backward_tiles_f64": (
        c_i32, [c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p,
                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "xg_backward_tiles": (
        c_i32,
        [c_i32, c_i32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size, c_void_p],
    ),
}

_lib = None


def load_library() -> ctypes.CDLL:
    """Load (building first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build

    try:
        stale = _build.needs_build()
    except OSError:
        stale = not LIB_PATH.exists()
    if stale and (os.environ.get("XG_NO_AUTOBUILD") != "1"):
        try:
            _build.build()
        except (OSError, RuntimeError) as exc:
            if not LIB_PATH.exists():
                raise NativeError(f"libxgauss.so is not built and the build failed: {exc}") from exc
    if not LIB_PATH.exists():
        raise NativeError(
            f"{LIB_PATH} missing: build it with `python -m paper_2403_04116_b200._build` "
            "(the engine has no CPU fallback)"
        )
    path = LIB_PATH
    variant = os.environ.get("XG_LIB_VARIANT")  # development: a tuning build (tools/variants.py)
    if variant:
        path = _build.variant_path(variant)
        if not path.exists():
            raise NativeError(f"variant library {path} not built")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.xg_abi_version() != XG_ABI_VERSION:
        raise NativeError("libxgauss ABI version mismatch")
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


def check(status: int, what: str) -> None:
    if status != XG_OK:
        msg = lib().xg_last_error().decode(errors="replace")
        if status == 1:
            raise InvalidParameterError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (status {status}): {msg}")


def require_cuda(t: torch.Tensor, name: str = "tensor") -> None:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise NativeError(
            f"{name} must be a CUDA tensor: the DRR engine runs only on the GPU (no CPU fallback)"
        )


def ptr(t: torch.Tensor | None, name: str = "tensor") -> int | None:
    if t is None:
        return None
    require_cuda(t, name)
    if not t.is_contiguous():
        raise InvalidParameterError(f"{name} must be contiguous")
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def cloud_struct(cloud, intensities: torch.Tensor | None = None,
                 invariants: torch.Tensor | None = None) -> XgCloud:
    s = XgCloud()
    s.params = ptr(cloud.flat, "cloud")
    s.basis = ptr(cloud.basis_weights, "basis_weights")
    s.n = cloud.n_points
    s.n_features = cloud.n_features
    s.intensities = ptr(intensities, "intensities")
    s.invariants = ptr(invariants, "invariants")
    return s


def raise_for_status(word: int, where: str = "") -> None:
    """Map device status bits onto the reference's exceptions, in the
    reference's check order (gaussians.py:56-57, frontend.py:134-136,
    gaussians.py:122-123, trainer.py:160-162)."""
    if word & XG_ST_ZERO_QUAT:
        raise InvalidParameterError("zero quaternion")
    if word & XG_ST_DEGENERATE:
        raise NumericalDegeneracyError("projected covariance not positive definite")
    if word & XG_ST_NONFINITE_FEAT:
        raise InvalidParameterError("feature and weights must be finite")
    if word & XG_ST_PEER_TIMEOUT:
        raise NativeError("peer gradient exchange timed out (a rank stopped stepping)")
    grad = (word >> XG_ST_GRAD_SHIFT) & 0x1F
    if grad:
        for f, name in enumerate(PARAM_FIELDS):
            if grad & (1 << f):
                raise TrainingDivergenceError(name)


def kernel_launches() -> int:
    return int(lib().xg_kernel_launches())


def view_invariants(cloud) -> torch.Tensor:
    """[N, 8] float64 view-independent projection terms (Sigma3, opacity,
    zero-quaternion flag) for a sweep over a static cloud (xg_view_invariants)."""
    out = torch.empty((cloud.n_points, 8), dtype=torch.float64, device=cloud.device)
    cs = cloud_struct(cloud)
    check(lib().xg_view_invariants(ctypes.byref(cs), ptr(out), stream()), "xg_view_invariants")
    return out


def intensities(cloud) -> torch.Tensor:
    out = torch.empty(cloud.n_points, dtype=torch.float32, device=cloud.device)
    counters = torch.zeros(XG_NCOUNTERS, dtype=torch.int32, device=cloud.device)
    cs = cloud_struct(cloud)
    check(lib().xg_intensities(ctypes.byref(cs), ptr(out), ptr(counters), stream()), "xg_intensities")
    raise_for_status(int(counters[XG_CTR_STATUS].item()))
    return out
