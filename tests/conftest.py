"""Shared fixtures.  ``gpu`` marks tests that need a CUDA device (run on the
B200 box with ``pytest -m gpu``); everything else runs on CPU."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libxgauss.so")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN, allow_pickle=False)
    return {k: data[k] for k in data.files}


def scene_names(g):
    return [str(s) for s in g["scenes"]]


def scene_fields(g, name):
    p = name + "/"
    return {f: g[p + f] for f in ("positions", "rotations", "log_scales", "raw_opacities", "features")}


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def small_scanner(width=16, height=16, pitch=12.0, n_views=4):
    """conftest.py:8-16 of the reference."""
    from paper_2403_04116_b200.geometry import ScannerConfig, equal_interval_angles

    return ScannerConfig(1000.0, 1500.0, width, height, pitch, equal_interval_angles(n_views))


def random_arrays(n, rng, n_features=4, pos_scale=40.0, scale_range=(3.0, 10.0), opacity_range=(0.05, 0.5)):
    """Same draws as the reference's random_cloud (conftest.py:19-40)."""
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    alphas = rng.uniform(*opacity_range, size=n)
    return {
        "positions": rng.uniform(-pos_scale, pos_scale, size=(n, 3)),
        "rotations": q,
        "log_scales": np.log(rng.uniform(*scale_range, size=(n, 3))),
        "raw_opacities": np.log(alphas) - np.log1p(-alphas),
        "features": rng.normal(scale=0.5, size=(n, n_features)),
    }


def normwise_ok(a, b, floor_scale, tol=1e-4):
    """max|a-b| <= tol * max(||b||_inf, floor_scale) (SURVEY 8c gradient metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return True, 0.0
    err = float(np.abs(a - b).max())
    scale = max(float(np.abs(b).max()), floor_scale)
    return err <= tol * scale, err / scale if scale > 0 else err
