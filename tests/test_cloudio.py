"""PLY checkpoint interchange with the reference (cloudio.py:1-108): a file
written by xsplat loads bit-exactly, and the same cloud saved here is
byte-identical to xsplat's file."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2403_04116_b200.cloudio import load_cloud, save_cloud
from paper_2403_04116_b200.errors import DatasetError

REF = Path(__file__).resolve().parent / "golden" / "ref_cloud.ply"


def test_reference_file_round_trips_byte_identical(tmp_path):
    c = load_cloud(REF)
    assert c.n_points == 40 and c.n_features == 5
    out = tmp_path / "mine.ply"
    save_cloud(c, out)
    assert out.read_bytes() == REF.read_bytes()


def test_truncated_and_foreign_files_raise(tmp_path):
    blob = REF.read_bytes()
    (tmp_path / "t.ply").write_bytes(blob[:-8])
    with pytest.raises(DatasetError):
        load_cloud(tmp_path / "t.ply")
    (tmp_path / "x.ply").write_bytes(b"not a ply")
    with pytest.raises(DatasetError):
        load_cloud(tmp_path / "x.ply")


def test_values_are_float32_exact():
    c = load_cloud(REF).to_numpy()
    for k in ("positions", "rotations", "log_scales", "raw_opacities", "features"):
        v = np.asarray(c[k], np.float64)
        assert np.array_equal(v, v.astype(np.float32).astype(np.float64)), k


def test_header_and_body_rules_match_reference(tmp_path):
    """cloudio.py:90-96 of the reference: a header without basis_weights is a
    DatasetError; a body longer than the vertices need is accepted."""
    blob = REF.read_bytes()
    pos = blob.find(b"end_header\n")
    hdr = b"\n".join(ln for ln in blob[:pos].split(b"\n") if not ln.startswith(b"comment basis_weights"))
    (tmp_path / "nw.ply").write_bytes(hdr + b"end_header\n" + blob[pos + len(b"end_header\n"):])
    with pytest.raises(DatasetError):
        load_cloud(tmp_path / "nw.ply")
    (tmp_path / "long.ply").write_bytes(blob + b"\0" * 24)
    a, b = load_cloud(tmp_path / "long.ply").to_numpy(), load_cloud(REF).to_numpy()
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
