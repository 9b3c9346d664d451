"""Helpers for tests/golden/fullsize.npz - the real reference's outputs at
BASELINE.json's full sizes (tests/golden/make_golden_fullsize.py).  Shared by
the CPU oracle pin (test_oracle_fullsize.py) and the GPU parity tests
(test_gpu_fullsize.py)."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

FULLSIZE = Path(__file__).resolve().parent / "golden" / "fullsize.npz"
PARAM_FIELDS = ("positions", "rotations", "log_scales", "raw_opacities", "features")
G_OF = {"C1": 68, "C2": 88, "C3": 152, "C4": 196}

_cache: dict = {}


def load() -> dict:
    if "fx" not in _cache:
        data = np.load(FULLSIZE, allow_pickle=False)
        _cache["fx"] = {k: data[k] for k in data.files}
    return _cache["fx"]


def cases() -> list[str]:
    return sorted({k.split("/")[0] for k in load() if "/" in k})


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cloud_arrays(case: str) -> dict:
    """The engine's own ACUI generator (acui.init_alternative_arrays) at the
    case's G, float32 - checked against the digest of the reference
    generator's cloud."""
    g = G_OF[case.split("_")[0]]
    key = ("cloud", g)
    if key not in _cache:
        from paper_2403_04116_b200 import acui

        arrs = acui.init_alternative_arrays("cuboid", acui.benchmark_spec(g), 16, 0)
        arrs = {k: np.ascontiguousarray(np.asarray(arrs[k], np.float32)) for k in PARAM_FIELDS}
        h = hashlib.sha256()
        for f in PARAM_FIELDS:
            h.update(arrs[f].tobytes())
        _cache[key] = (arrs, h.hexdigest())
    arrs, digest = _cache[key]
    assert digest == str(load()[case + "/cloud_sha"]), f"{case}: engine ACUI cloud != reference generator's"
    return arrs


def camera(case: str):
    l_so, l_sd, w, h, pitch, phi = load()[case + "/camera"]
    return float(l_so), float(l_sd), int(w), int(h), float(pitch), float(phi)


def ref_form(entry_ids: np.ndarray, active: np.ndarray, n: int) -> np.ndarray:
    """Cloud-index entry list -> the reference's active-row form
    (frontend.py:166-170: entry_splat holds rows of active_indices)."""
    row = np.full(n, -1, dtype=np.int64)
    row[active] = np.arange(active.size)
    return row[np.asarray(entry_ids, np.int64)].astype(np.int32)


def check_binning(case: str, active: np.ndarray, entry_splat_rows: np.ndarray, tile_ranges: np.ndarray,
                  depths: np.ndarray) -> None:
    """Bit-exact comparison with the reference's SplatList; on an entry
    mismatch, names the first differing tiles."""
    fx = load()
    p = case + "/"
    assert sha(np.asarray(active, np.int64)) == str(fx[p + "active_sha"]), f"{case}: active set"
    assert np.array_equal(tile_ranges, fx[p + "tile_ranges"]), f"{case}: tile ranges"
    assert sha(np.asarray(depths, np.float64)) == str(fx[p + "depths_sha"]), f"{case}: float64 depths"
    es = np.ascontiguousarray(entry_splat_rows, np.int32)
    if sha(es) != str(fx[p + "entry_sha"]):
        bad = []
        for t, (a, b) in enumerate(fx[p + "tile_ranges"]):
            d = np.frombuffer(hashlib.blake2b(es[a:b].tobytes(), digest_size=8).digest(), np.uint64)[0]
            if d != fx[p + "tile_sha"][t]:
                bad.append(t)
        raise AssertionError(f"{case}: entry order differs from the reference in {len(bad)} tiles: {bad[:10]}")
