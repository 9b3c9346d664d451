"""CPU checks of the drop-in boundary: libxgauss.so loads (no GPU needed) and
exports exactly what include/xgauss.h declares; the ctypes binding covers it."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_functions() -> set[str]:
    text = (ROOT / "include" / "xgauss.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(xg_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_entry_points():
    names = declared_functions()
    for must in ("xg_preprocess_fwd", "xg_bin_sort", "xg_composite_fwd", "xg_composite_bwd",
                 "xg_preprocess_bwd", "xg_adam", "xg_densify_mark", "xg_densify_apply",
                 "xg_forward_tiles", "xg_backward_tiles", "xg_bin_workspace_bytes"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    from paper_2403_04116_b200 import _native

    lib = _native.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.xg_abi_version() == _native.XG_ABI_VERSION == 5


def test_binding_covers_header():
    from paper_2403_04116_b200 import _native

    assert declared_functions() == set(_native.SIGNATURES)


def test_workspace_queries_without_gpu():
    from paper_2403_04116_b200 import _native

    lib = _native.load_library()
    assert lib.xg_bin_workspace_bytes(1000, 20000, 16) > 8 * 1000
    assert lib.xg_tiles_workspace_bytes(100, 64, 64) > 4 * 64 * 64
    assert lib.xg_densify_scratch_bytes(1000) >= 4 * 6 * 1000


def test_invalid_arguments_are_rejected_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_2403_04116_b200 import _native

    lib = _native.load_library()
    assert lib.xg_preprocess_fwd(None, None, None, None, None) == 1
    assert b"invalid" in lib.xg_last_error()
    assert lib.xg_adam(None, None, None, None, 0, 0, None, 0.9, 0.999, 1e-15, 1.0, 1.0, None, None) == 1


def test_no_cpu_fallback():
    """Rendering a CPU-resident cloud fails loudly instead of falling back."""
    import numpy as np
    import pytest

    import paper_2403_04116_b200 as xg
    from paper_2403_04116_b200.errors import NativeError

    cloud = xg.GaussianCloud(np.zeros((1, 3)), [[1.0, 0, 0, 0]], np.zeros((1, 3)), [0.0], np.zeros((1, 2)),
                             device="cpu")
    sc = xg.ScannerConfig(1000.0, 1500.0, 16, 16, 12.0)
    with pytest.raises(NativeError):
        xg.render_view(cloud, sc, 0.0)
    _ = ctypes
