"""CPU checks of the phantom / dataset host layer against golden vectors of
the real reference (tests/golden/make_golden_phantom.py): voxelisation,
noise draw, and the on-disk format (dataset.py:118-192) round trip."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2403_04116_b200 import dataset as ds
from paper_2403_04116_b200 import phantom as pm
from paper_2403_04116_b200.errors import DatasetError, InvalidParameterError
from paper_2403_04116_b200.geometry import ScannerConfig, equal_interval_angles

GOLD = Path(__file__).resolve().parent / "golden" / "phantom.npz"


@pytest.fixture(scope="module")
def gold():
    d = np.load(GOLD, allow_pickle=False)
    return {k: d[k] for k in d.files}


def test_voxelisation_matches_reference(gold):
    grid, vs = tuple(int(v) for v in gold["A/grid"]), gold["A/voxel_size"]
    ph = pm.make_phantom(pm.default_phantom_primitives(np.array(grid) * vs), grid, vs)
    assert np.array_equal(ph.densities, gold["A/densities"])
    g = int(gold["B/g"])
    phb = pm.make_phantom(pm.default_phantom_primitives(np.full(3, 200.0)), (g, g, g), np.full(3, 200.0 / g))
    assert phb.densities.sum() == float(gold["B/density_sum"])
    assert int((phb.densities > 0).sum()) == int(gold["B/density_nnz"])
    phc = pm.make_phantom([pm.Cuboid([0.0, 0.0, 0.0], [16.0, 16.0, 16.0], 0.5),
                           pm.Ellipsoid([8.0, -8.0, 0.0], [8.0, 8.0, 8.0], 0.25)], (16, 16, 16), np.full(3, 2.0))
    assert np.array_equal(phc.densities, gold["C/densities"])


def test_primitive_validation_and_dicts():
    with pytest.raises(InvalidParameterError):
        pm.Ellipsoid([0, 0, 0], [1, 0, 1], 1.0)
    with pytest.raises(InvalidParameterError):
        pm.Cuboid([0, 0, 0], [1, 1, 1], -1.0)
    with pytest.raises(InvalidParameterError):
        pm.make_phantom([pm.Cuboid([0, 0, 0], [20, 1, 1], 1.0)], (4, 4, 4), 2.0)
    with pytest.raises(InvalidParameterError):
        pm.primitive_from_dict({"kind": "torus"})
    for p in pm.default_phantom_primitives(np.full(3, 100.0)):
        q = pm.primitive_from_dict(p.to_dict())
        assert type(q) is type(p) and q.to_dict() == p.to_dict()


def test_noise_matches_reference(gold):
    sc = ScannerConfig(1000.0, 1500.0, 48, 40, 6.0, equal_interval_angles(4))
    imgs = gold["A/images"]
    tr, te = ds.alternating_split(4)
    ps = ds.ProjectionSet(imgs, imgs.copy(), sc, tr, te, float(gold["A/normalization"]))
    noisy = ds.add_noise(ps, 0.03, 0)
    assert np.array_equal(noisy.images, gold["A/noisy"])
    assert np.array_equal(noisy.clean_images, imgs)
    assert ds.add_noise(ps, 0.0).images is not None
    with pytest.raises(InvalidParameterError):
        ds.add_noise(ps, -1.0)


def test_save_load_round_trip(gold, tmp_path):
    sc = ScannerConfig(1000.0, 1500.0, 48, 40, 6.0, equal_interval_angles(4))
    imgs = gold["A/images"]
    tr, te = ds.alternating_split(4)
    ps = ds.add_noise(ds.ProjectionSet(imgs, imgs.copy(), sc, tr, te, 2.5, phantom_spec={"grid": [1, 2, 3]}),
                      0.03, 7)
    ds.save_dataset(ps, tmp_path / "set")
    back = ds.load_dataset(tmp_path / "set")
    assert np.array_equal(back.images, ps.images) and np.array_equal(back.clean_images, ps.clean_images)
    assert np.array_equal(back.angles, ps.angles)
    assert back.normalization == 2.5 and back.noise_seed == 7 and back.phantom_spec == {"grid": [1, 2, 3]}
    assert np.array_equal(back.train_indices, tr) and np.array_equal(back.test_indices, te)
    (tmp_path / "set" / "proj_0003.f32").write_bytes(b"\0" * 12)
    with pytest.raises(DatasetError):
        ds.load_dataset(tmp_path / "set")
    with pytest.raises(DatasetError):
        ds.load_dataset(tmp_path / "missing")
