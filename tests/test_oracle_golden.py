"""The CPU oracle (oracle/swsdc_oracle.py) pinned against golden vectors that
the REFERENCE produced (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

import swsdc_oracle as orc
from conftest import GOLDEN, TEST_PARAMS, rel_err

from paper_1805_07923_b200 import workloads


@pytest.fixture(scope="module")
def gt():
    return np.load(os.path.join(GOLDEN, "transforms.npz"))


@pytest.fixture(scope="module")
def gr():
    return np.load(os.path.join(GOLDEN, "rhs.npz"))


def test_gauss_nodes_bitwise():
    g = np.load(os.path.join(GOLDEN, "grids.npz"))
    for n in (1, 2, 3, 7, 24, 47, 48, 96, 128, 191, 192, 384):
        mu, w = orc.gauss_nodes(n)
        np.testing.assert_array_equal(mu, g[f"mu_{n}"])
        np.testing.assert_array_equal(w, g[f"w_{n}"])


CASES = [(31, 96, 47), (31, 96, 48), (15, 48, 24), (10, 33, 17), (63, 192, 96)]


@pytest.mark.parametrize("R,I,J", CASES)
def test_oracle_transforms(gt, R, I, J):
    tag = f"R{R}_I{I}_J{J}"
    p = orc.OraclePlan(R, I, J)
    assert rel_err(p.synthesize(gt[f"{tag}_c"]), gt[f"{tag}_syn"]) < 1e-13
    assert rel_err(p.analyze(gt[f"{tag}_g"]), gt[f"{tag}_ana"]) < 1e-13
    u, v = p.synth_uv(gt[f"{tag}_c"], gt[f"{tag}_c2"])
    assert rel_err(u, gt[f"{tag}_u"]) < 1e-13 and rel_err(v, gt[f"{tag}_v"]) < 1e-13
    d, k = p.anal_divcurl(gt[f"{tag}_g"], gt[f"{tag}_g2"])
    assert rel_err(d, gt[f"{tag}_div"]) < 1e-13 and rel_err(k, gt[f"{tag}_curl"]) < 1e-13
    assert rel_err(p.to_fourier(gt[f"{tag}_g"]), gt[f"{tag}_fourier"]) < 1e-14
    if f"{tag}_P" in gt:
        np.testing.assert_array_equal(p.P, gt[f"{tag}_P"])
        np.testing.assert_array_equal(p.H, gt[f"{tag}_H"])


@pytest.mark.parametrize("R,I,J", [(15, 48, 24), (31, 96, 47), (31, 96, 48)])
def test_oracle_rhs(gr, R, I, J):
    tag = f"R{R}_I{I}_J{J}"
    prm = orc.OracleParams(**TEST_PARAMS)
    x = gr[f"{tag}_x"]
    for nl in (True, False):
        rhs = orc.OracleRHS(orc.OraclePlan(R, I, J), prm, nl)
        got = rhs.eval_fe(x)
        want = gr[f"{tag}_fe_nl{int(nl)}"]
        for f in range(3):
            assert rel_err(got[f], want[f]) < 1e-12
    rhs = orc.OracleRHS(orc.OraclePlan(R, I, J), prm)
    np.testing.assert_allclose(rhs.eval_fi(x), gr[f"{tag}_fi"], rtol=0, atol=0)
    for beta in (0.0, 112.5, 600.0):
        np.testing.assert_array_equal(rhs.solve(x, beta), gr[f"{tag}_solve_{beta}"])


def test_oracle_sweeps():
    g = np.load(os.path.join(GOLDEN, "sweeps.npz"))
    prm = orc.OracleParams(**workloads.EARTH)
    for n_nodes, dt in ((3, 600.0), (5, 450.0)):
        lvl = orc.OracleLevel(15, n_nodes, prm)
        y = orc.sdc_step(g[f"sdc{n_nodes}_x"], dt, 2, lvl.tb, lvl.rhs)
        assert rel_err(y, g[f"sdc{n_nodes}_out"]) < 1e-12
    for nf, nc, ncs, dt in ((3, 2, 1, 600.0), (5, 3, 2, 240.0)):
        h = orc.OracleHierarchy(orc.OracleLevel(31, nf, prm, (96, 48)),
                                orc.OracleLevel(15, nc, prm, (48, 24)))
        tag = f"ml{nf}{nc}_cs{ncs}"
        y = orc.mlsdc_step(g[f"{tag}_x"], dt, 2, h, ncs)
        assert rel_err(y, g[f"{tag}_out"]) < 1e-12
        r = [h.fine.rhs.n_solve, h.fine.rhs.n_fi, h.fine.rhs.n_fe, h.coarse.rhs.n_solve,
             h.coarse.rhs.n_fi, h.coarse.rhs.n_fe]
        assert r == list(g[f"{tag}_counts"])


def test_oracle_config0():
    g = np.load(os.path.join(GOLDEN, "config0.npz"))
    prm = orc.OracleParams(**workloads.EARTH)
    h = orc.OracleHierarchy(orc.OracleLevel(63, 3, prm, (192, 96)),
                            orc.OracleLevel(31, 2, prm, (96, 48)))
    y = orc.mlsdc_step(g["x"], 600.0, 2, h)
    for f in range(3):
        assert rel_err(y[f], g["out"][f]) < 1e-12


def test_oracle_errors():
    with pytest.raises(ValueError):
        orc.gauss_nodes(0)
    with pytest.raises(ValueError):
        orc.OraclePlan(-1, 8, 4)
    with pytest.raises(ValueError):
        orc.OraclePlan(10, 20, 16)
    p = orc.OraclePlan(7, 24, 12)
    with pytest.raises(ValueError):
        p.analyze(np.zeros((4, 4)))
    with pytest.raises(ValueError):
        p.synthesize(np.zeros((10, 10), dtype=complex))
    with pytest.raises(ValueError):
        orc.lobatto(4)
    rhs = orc.OracleRHS(p, orc.OracleParams())
    with pytest.raises(ValueError):
        rhs.solve(np.zeros((3, 8, 8), dtype=complex), -1.0)
