"""Host-side logic of the product package and the C ABI, on the CPU."""

import ctypes
import os
import re

import numpy as np
import pytest

import swsdc_oracle as orc
from conftest import GOLDEN, ROOT

from paper_1805_07923_b200 import _lib, workloads


def test_host_gauss_nodes_bitwise_vs_reference():
    from paper_1805_07923_b200 import spharm
    g = np.load(os.path.join(GOLDEN, "grids.npz"))
    for n in (1, 2, 3, 7, 24, 47, 48, 96, 128, 191, 192, 384):
        mu, w = spharm.gauss_legendre_nodes(n)
        np.testing.assert_array_equal(mu, g[f"mu_{n}"])
        np.testing.assert_array_equal(w, g[f"w_{n}"])
    with pytest.raises(ValueError):
        spharm.gauss_legendre_nodes(0)


def test_grid_shapes():
    from paper_1805_07923_b200 import spharm
    assert spharm.next_fast_size(190) == 192
    assert spharm.next_fast_size(97) == 100
    assert spharm.default_grid_shape(31) == orc.default_shape(31) == (96, 47)
    assert spharm.default_grid_shape(63) == (192, 95)
    grid = spharm.build_gaussian_grid(24)
    assert np.all(np.diff(grid.mu) > 0)
    np.testing.assert_array_equal(grid.mu, -grid.mu[::-1])
    assert abs(grid.w.sum() - 2.0) < 1e-12


def test_sdc_tables_match_oracle_and_known_answers():
    from paper_1805_07923_b200 import mlsdc, sdc
    for n in (2, 3, 5):
        t = sdc.build_tables(n)
        o = orc.OracleTables(n)
        np.testing.assert_array_equal(t.q, o.q)
        np.testing.assert_array_equal(t.q_delta_i, o.qi)
        np.testing.assert_array_equal(t.q_delta_e, o.qe)
    # reference test_sdc.py:101-106 hand LU for 3 nodes
    np.testing.assert_allclose(sdc.build_tables(3).q_delta_i,
                               [[0, 0, 0], [0, 1 / 3, 0], [0, 2 / 3, 1 / 4]], atol=1e-14)
    with pytest.raises(ValueError):
        sdc.lobatto_nodes(4)
    with pytest.raises(RuntimeError):
        sdc._lu_nopivot(np.array([[0.0, 1.0], [1.0, 0.0]]))
    pi = mlsdc.time_transfer_matrix(sdc.lobatto_nodes(5), sdc.lobatto_nodes(3))
    for row in pi:
        assert sorted(row) == [0.0] * 4 + [1.0]
    with pytest.raises(ValueError):
        mlsdc.TransferOps.build(sdc.lobatto_nodes(3), sdc.lobatto_nodes(5), 31, 15)


def test_seeded_inputs_follow_recipe():
    st = workloads.seeded_state(31, 0)
    mult = np.full((32, 1), 2.0)
    mult[0] = 1.0
    for f, tgt in enumerate(workloads.RMS_TARGETS):
        rms = np.sqrt(np.sum(mult * np.abs(st[f]) ** 2) / 2.0)
        assert abs(rms / tgt - 1.0) < 1e-12
        assert np.all(st[f][0].imag == 0.0)
        assert np.all(np.tril(st[f], -1) == 0.0)
    assert st[1][0, 0] == 0.0 and st[2][0, 0] == 0.0
    np.testing.assert_array_equal(workloads.seeded_state(31, 0), st)
    # the grid rms of the oracle synthesis equals the target (Parseval)
    p = orc.OraclePlan(31, 96, 48)
    g = p.synthesize(st[0])
    rms_grid = np.sqrt(np.sum(g * g * p.w) / (2.0 * p.I))
    assert abs(rms_grid / 1e3 - 1.0) < 1e-12


def test_c_abi_exports_every_declared_symbol():
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "swsdc_b200.h")).read()
    declared = set(re.findall(r"\b(swsdc_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED_SYMBOLS) == declared
    assert lib.swsdc_version().startswith(b"swsdc_b200")


@pytest.mark.parametrize("R,nmat", [(0, 1), (5, 3), (63, 7), (255, 15)])
def test_pack_triangles_host(R, nmat):
    """Host half of the packed upload: the s >= r triangles row after row, whatever the
    slicing over the packing threads (T255 x 15 is the config-1 batch: 16 slices)."""
    lib = _lib.load()
    rng = np.random.default_rng(R)
    dense = rng.standard_normal((nmat, R + 1, R + 1)) + 1j * rng.standard_normal((nmat, R + 1, R + 1))
    tri = np.triu_indices(R + 1)
    packed = np.full((nmat, len(tri[0])), np.nan + 0j)
    for _ in range(2):
        assert lib.swsdc_pack_triangles(dense.ctypes.data_as(ctypes.c_void_p), R, nmat,
                                        packed.ctypes.data_as(ctypes.c_void_p)) == 0
        np.testing.assert_array_equal(packed, dense[:, tri[0], tri[1]])
    assert lib.swsdc_pack_triangles(None, R, nmat, None) == 1
    assert lib.swsdc_pack_triangles(None, R, 0, None) == 0


def test_c_abi_usage_errors_need_no_gpu():
    lib = _lib.load()
    mu = np.zeros(8)
    h = ctypes.c_void_p()
    p = mu.ctypes.data_as(ctypes.c_void_p)
    assert lib.swsdc_plan_create(-1, 16, 8, p, p, ctypes.byref(h)) == 1
    with pytest.raises(ValueError, match="non-negative"):
        _lib.check(1)
    assert lib.swsdc_plan_create(10, 20, 8, p, p, ctypes.byref(h)) == 1
    assert b"cannot carry" in lib.swsdc_last_error()
    assert lib.swsdc_plan_create(3, 17 * 19, 8, p, p, ctypes.byref(h)) == 1
    prm = _lib.Params(6.37e6, 7.292e-5, 9.8, 1e5, 1e4)
    assert lib.swsdc_solve_implicit(3, ctypes.byref(prm), -1.0, None, 0, None, None) == 1
    bad = _lib.Params(6.37e6, 7.292e-5, 9.8, -1.0, 1e4)
    assert lib.swsdc_eval_fi(3, ctypes.byref(bad), None, 0, None, None) == 1
    # the singular-determinant check is host-side (implicit.py:332-333)
    big = _lib.Params(1.0, 7.292e-5, 9.8, 0.0, 1e4)
    assert lib.swsdc_solve_implicit(3, ctypes.byref(big), 1e3, None, 0, None, None) in (0, 2)
