"""Deflation-vector construction: labels, column map and d bit-exact with the reference.

CPU tests pin the oracle's labellers (oracle/dk_oracle.py) to the reference's own outputs
(tests/golden, written by make_golden.py from physics.py:119-143 as shipped); GPU tests pin
the product's device labeller (dk_levelset_labels_device) to the same goldens and to the
oracle on random fields.  The product has no host labeller: without a device the partition
API raises DeviceUnavailable.
"""
from __future__ import annotations

import zlib

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import _lib, configs
from oracle import dk_oracle as O

BIG = [(2, "config2"), (3, "config3_labels"), (4, "config4_labels"), (5, "config5_labels")]


def crc64(labels) -> int:
    return zlib.crc32(np.ascontiguousarray(np.asarray(labels).astype(np.int64)).tobytes())


def hetero_field(g):
    grid = dk.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    return dk.PermeabilityField(grid, g["kx"], g["ky"], g["kz"])


def sandwich_field():
    return dk.make_layered_field(dk.Grid(7, 7, 3), [((0, 1), 1e6), ((1, 2), 1.0), ((2, 3), 1e6)])


# ---- oracle against the reference (CPU) -------------------------------------------------
@pytest.mark.parametrize("labeller", [O.subdomain_levelset_labels,
                                      O.subdomain_levelset_labels_boxwise])
def test_oracle_labels_hetero_sandwich_config1(golden, labeller):
    g = golden("hetero")
    lab, d, excl = labeller(g["kx"], 12, 10, 8, 3, 2, 2, 1.0)
    np.testing.assert_array_equal(lab, g["labels"])
    assert d == int(g["d"]) and sorted(excl) == list(g["excl"]) and len(excl) > 0
    s = golden("sandwich")
    lab, d, _ = labeller(sandwich_field().kx, 7, 7, 3, 1, 1, 1, 2.0)
    np.testing.assert_array_equal(lab, s["labels"])
    c = configs.config1()
    lab, d, _ = labeller(c.band_field.kx, 32, 32, 32, 2, 2, 2, 2.0)
    np.testing.assert_array_equal(lab, golden("config1")["labels"])
    assert d == 16


@pytest.mark.parametrize("idx,name", BIG)
def test_oracle_labels_full_size_crc(golden, idx, name):
    """BASELINE configs 2-5 at full size: the oracle's box-wise labeller reproduces the
    reference partition's d, excluded ids and label-vector CRC (config 5: 67 M cells)."""
    g = golden(name)
    c = configs.make_case(idx)
    gr = c.grid
    lab, d, excl = O.subdomain_levelset_labels_boxwise(c.band_field.kx, gr.nx, gr.ny, gr.nz,
                                                       *c.boxes, c.jump_threshold)
    assert d == int(g["d"])
    assert crc64(lab) == int(g["labels_crc"])
    if "sizes" in g:
        np.testing.assert_array_equal(np.bincount(lab, minlength=d), g["sizes"])
        assert sorted(excl) == list(g["excl"])


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 2**31 - 1), st.integers(1, 4), st.integers(1, 3), st.integers(1, 3),
       st.sampled_from([0.5, 1.0, 2.0]))
def test_boxwise_oracle_equals_full_grid_oracle(seed, px, py, pz, thr):
    rng = np.random.default_rng(seed)
    nx, ny, nz = rng.integers(px, 9), rng.integers(py, 7), rng.integers(pz, 6)
    n = nx * ny * nz
    kx = 10.0 ** rng.integers(-3, 3, n).astype(float)
    kx[rng.random(n) < 0.15] = 0.0
    a = O.subdomain_levelset_labels(kx, nx, ny, nz, px, py, pz, thr)
    b = O.subdomain_levelset_labels_boxwise(kx, nx, ny, nz, px, py, pz, thr)
    np.testing.assert_array_equal(a[0], b[0])
    assert a[1] == b[1] and a[2] == b[2]


# ---- host logic of the partition API (CPU) ------------------------------------------------
def test_partition_to_basis_column_map(golden):
    g = golden("hetero")
    p = dk.Partition(g["labels"], int(g["d"]), "subdomain_levelset",
                     frozenset(int(e) for e in g["excl"]))
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
    with pytest.raises(ValueError):
        dk.levelset_partition(dk.PermeabilityField(dk.Grid(2, 1, 1), np.array([1.0, -1.0]),
                                                   np.ones(2), np.ones(2)))


def test_no_host_fallback_for_labels():
    """The partition builders run on the device only (no CPU fallback)."""
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(dk.DeviceUnavailable):
        dk.subdomain_levelset_partition(sandwich_field(), 1, 1, 1)
    with pytest.raises(dk.DeviceUnavailable):
        dk.subdomain_partition(dk.Grid(4, 4, 4), 2, 2, 2)


def test_manual_layers_and_files(tmp_path):
    grid = dk.Grid(2, 2, 4)
    p = dk.manual_layers(grid, [(0, 1), (2, 4)])
    assert p.d == 3 and p.default_exclude == frozenset({2})
    path = tmp_path / "part.txt"
    dk.save_partition(path, p)
    q = dk.load_partition(path)
    np.testing.assert_array_equal(q.labels, p.labels)


# ---- the device labeller against the reference (GPU) -----------------------------------
@pytest.mark.gpu
def test_device_labels_hetero_sandwich_config1(gpu, golden):
    g = golden("hetero")
    p = dk.subdomain_levelset_partition(hetero_field(g), 3, 2, 2, 1.0)
    np.testing.assert_array_equal(p.labels, g["labels"])
    assert p.d == int(g["d"]) and sorted(p.default_exclude) == list(g["excl"])
    p = dk.levelset_partition(sandwich_field(), 2.0)
    np.testing.assert_array_equal(p.labels, golden("sandwich")["labels"])
    assert p.d == 3
    p = configs.config1().partition()
    np.testing.assert_array_equal(p.labels, golden("config1")["labels"])
    assert p.d == 16


@pytest.mark.gpu
@pytest.mark.parametrize("idx,name", BIG)
def test_device_labels_full_size_crc(gpu, golden, idx, name):
    """BASELINE configs 2-5: d, excluded ids and the label CRC of the reference partition."""
    g = golden(name)
    p = configs.make_case(idx).partition()
    assert p.d == int(g["d"])
    assert crc64(p.labels) == int(g["labels_crc"])
    if "sizes" in g:
        assert sorted(p.default_exclude) == list(g["excl"])


@pytest.mark.gpu
@settings(max_examples=30, deadline=None)
@given(st.integers(0, 2**31 - 1), st.integers(1, 4), st.integers(1, 3), st.integers(1, 3),
       st.sampled_from([0.5, 1.0, 2.0]))
def test_device_labels_random_fields_match_oracle(gpu, seed, px, py, pz, thr):
    rng = np.random.default_rng(seed)
    nx, ny, nz = rng.integers(px, 17), rng.integers(py, 11), rng.integers(pz, 9)
    n = nx * ny * nz
    kx = 10.0 ** rng.integers(-3, 3, n).astype(float)
    kx[rng.random(n) < 0.15] = 0.0
    f = dk.PermeabilityField(dk.Grid(int(nx), int(ny), int(nz)), kx, kx, kx)
    p = dk.subdomain_levelset_partition(f, px, py, pz, thr)
    lab, d, excl = O.subdomain_levelset_labels(kx, nx, ny, nz, px, py, pz, thr)
    np.testing.assert_array_equal(p.labels, lab)
    assert p.d == d and set(p.default_exclude) == excl


@pytest.mark.gpu
def test_device_subdomain_partition_remainders(gpu):
    p = dk.subdomain_partition(dk.Grid(7, 5, 3), 3, 2, 1)
    assert p.d == 6
    lab = p.labels.reshape(3, 5, 7)
    # nc // p with the remainder to the leading blocks: x sizes 3, 2, 2
    assert list(lab[0, 0]) == [0, 0, 0, 1, 1, 2, 2]
