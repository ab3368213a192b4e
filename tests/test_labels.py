"""Deflation-vector construction: labels, column map and d bit-exact with the reference."""
from __future__ import annotations

import zlib

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
from oracle import dk_oracle as O


def test_hetero_subdomain_levelset(golden):
    g = golden("hetero")
    grid = dk.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    f = dk.PermeabilityField(grid, g["kx"], g["ky"], g["kz"])
    p = dk.subdomain_levelset_partition(f, 3, 2, 2, 1.0)
    np.testing.assert_array_equal(p.labels, g["labels"])
    assert p.d == int(g["d"])
    assert sorted(p.default_exclude) == list(g["excl"])
    assert len(p.default_exclude) > 0  # the field has zero-permeability components


def test_sandwich_levelset(golden):
    g = golden("sandwich")
    grid = dk.Grid(7, 7, 3)
    f = dk.make_layered_field(grid, [((0, 1), 1e6), ((1, 2), 1.0), ((2, 3), 1e6)])
    p = dk.levelset_partition(f, 2.0)
    np.testing.assert_array_equal(p.labels, g["labels"])
    assert p.d == 3


def test_config1_labels(golden):
    g = golden("config1")
    p = configs.config1().partition()
    np.testing.assert_array_equal(p.labels, g["labels"])
    assert p.d == int(g["d"]) == 16


@pytest.mark.parametrize("idx,name", [(2, "config2"), (3, "config3_labels")])
def test_full_size_labels_crc(golden, idx, name):
    """Configs 2 and 3 at full size: d and a CRC of the reference's label vector."""
    g = golden(name)
    p = configs.make_case(idx).partition()
    assert p.d == int(g["d"])
    assert zlib.crc32(np.ascontiguousarray(p.labels.astype(np.int64)).tobytes()) == \
        int(g["labels_crc"])


@settings(max_examples=30, deadline=None)
@given(st.integers(0, 2**31 - 1), st.integers(1, 4), st.integers(1, 3), st.integers(1, 3),
       st.sampled_from([0.5, 1.0, 2.0]))
def test_random_fields_match_oracle(seed, px, py, pz, thr):
    rng = np.random.default_rng(seed)
    nx, ny, nz = rng.integers(px, 9), rng.integers(py, 7), rng.integers(pz, 6)
    n = nx * ny * nz
    kx = 10.0 ** rng.integers(-3, 3, n).astype(float)
    kx[rng.random(n) < 0.15] = 0.0
    grid = dk.Grid(int(nx), int(ny), int(nz))
    f = dk.PermeabilityField(grid, kx, kx, kx)
    p = dk.subdomain_levelset_partition(f, px, py, pz, thr)
    lab, d, excl = O.subdomain_levelset_labels(kx, nx, ny, nz, px, py, pz, thr)
    np.testing.assert_array_equal(p.labels, lab)
    assert p.d == d and set(p.default_exclude) == excl


def test_subdomain_partition_remainders():
    grid = dk.Grid(7, 5, 3)
    p = dk.subdomain_partition(grid, 3, 2, 1)
    assert p.d == 6
    lab = p.labels.reshape(3, 5, 7)
    # nc // p with the remainder to the leading blocks: x sizes 3, 2, 2
    assert list(lab[0, 0]) == [0, 0, 0, 1, 1, 2, 2]


def test_partition_to_basis_column_map(golden):
    g = golden("hetero")
    grid = dk.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    p = dk.subdomain_levelset_partition(dk.PermeabilityField(grid, g["kx"], g["ky"], g["kz"]),
                                        3, 2, 2, 1.0)
    B = dk.partition_to_basis(p)
    col, dd = O.columns_from_labels(p.labels, p.d, p.default_exclude)
    np.testing.assert_array_equal(B.labels, col)
    assert B.d == dd == p.d - len(p.default_exclude)
    B2 = dk.partition_to_basis(p, exclude_labels=[])
    assert B2.d == p.d and np.all(B2.labels >= 0)
    with pytest.raises(ValueError):
        dk.partition_to_basis(p, exclude_labels=range(p.d))


def test_partition_validation():
    with pytest.raises(ValueError):
        dk.Partition(np.array([0, 2]), 2, "manual")
    with pytest.raises(ValueError):
        dk.Partition(np.array([0, 0]), 2, "manual")
    with pytest.raises(ValueError):
        dk.subdomain_partition(dk.Grid(3, 3, 3), 4, 1, 1)
    with pytest.raises(ValueError):
        dk.levelset_partition(dk.make_layered_field(dk.Grid(2, 2, 2), [((0, 2), 1.0)]), 0.0)


def test_manual_layers_and_files(tmp_path):
    grid = dk.Grid(2, 2, 4)
    p = dk.manual_layers(grid, [(0, 1), (2, 4)])
    assert p.d == 3 and p.default_exclude == frozenset({2})
    path = tmp_path / "part.txt"
    dk.save_partition(path, p)
    q = dk.load_partition(path)
    np.testing.assert_array_equal(q.labels, p.labels)
