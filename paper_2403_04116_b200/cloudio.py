"""Cloud checkpoints in the reference's PLY layout (``cloudio.py:1-108``).

Binary little-endian PLY, one ``vertex`` per Gaussian with float64
properties ``x y z q0 q1 q2 q3 s0 s1 s2 raw_opacity f_0 .. f_{n-1}`` and the
header comments ``n_features`` / ``basis_weights`` (repr-exact), so files
interchange with xsplat in both directions.  The device cloud is float32
(parameters and basis weights): a float32-origin cloud round-trips save +
load bit for bit; a reference checkpoint's float64 values are rounded to
float32 on load, so re-saving it is bit-exact only where they were float32
values to begin with (``tests/test_cloudio.py``: a reference-written cloud of
float32 values re-saves byte-identically).  Validation follows
``cloudio.py:60-108``: a missing ``basis_weights`` comment is a
``DatasetError``, a body LONGER than the vertices need is accepted.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import DatasetError
from .gaussians import GaussianCloud


def _names(nf: int) -> list[str]:
    return ["x", "y", "z", "q0", "q1", "q2", "q3", "s0", "s1", "s2", "raw_opacity"] + [f"f_{k}" for k in range(nf)]


def save_cloud(cloud: GaussianCloud, path: str | os.PathLike) -> None:
    f = cloud.to_numpy()
    data = np.concatenate([f["positions"], f["rotations"], f["log_scales"], f["raw_opacities"][:, None],
                           f["features"]], axis=1)
    hdr = ["ply", "format binary_little_endian 1.0", f"comment n_features {cloud.n_features}",
           "comment basis_weights " + " ".join(repr(float(w)) for w in f["basis_weights"]),
           f"element vertex {cloud.n_points}"]
    hdr += [f"property double {n}" for n in _names(cloud.n_features)]
    hdr.append("end_header")
    with open(path, "wb") as fh:
        fh.write(("\n".join(hdr) + "\n").encode("ascii"))
        fh.write(np.ascontiguousarray(data, dtype="<f8").tobytes())


def load_cloud(path: str | os.PathLike, device=None) -> GaussianCloud:
    blob = open(path, "rb").read()
    if not blob.startswith(b"ply"):
        raise DatasetError(f"{path}: not a PLY file")
    pos = blob.find(b"end_header\n")
    if pos < 0:
        raise DatasetError(f"{path}: missing end_header")
    n = nf = None
    weights = None
    props = []
    for line in blob[:pos].decode("ascii").splitlines():
        p = line.split()
        if not p:
            continue
        if p[:2] == ["comment", "n_features"]:
            nf = int(p[2])
        elif p[:2] == ["comment", "basis_weights"]:
            weights = np.array([float(v) for v in p[2:]])
        elif p[:2] == ["element", "vertex"]:
            n = int(p[2])
        elif p[0] == "property":
            if p[1] != "double":
                raise DatasetError(f"{path}: unsupported property type {p[1]}")
            props.append(p[2])
    if n is None or nf is None or weights is None:
        raise DatasetError(f"{path}: header missing vertex count, n_features or basis_weights")
    if props != _names(nf):
        raise DatasetError(f"{path}: property list does not match the checkpoint schema")
    body = blob[pos + len(b"end_header\n"):]
    need = 8 * n * len(props)
    if len(body) < need:  # (trailing bytes are ignored, as the reference does)
        raise DatasetError(f"{path}: body holds {len(body)} bytes, expected {need}")
    data = np.frombuffer(body[:need], dtype="<f8").reshape(n, len(props))
    return GaussianCloud(data[:, 0:3], data[:, 3:7], data[:, 7:10], data[:, 10], data[:, 11:],
                         basis_weights=weights, device=device)
