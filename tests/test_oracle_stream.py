"""The streaming per-r oracle (oracle/swsdc_stream.py) -- CPU only.

Pinned three ways: its tables are bitwise the dense oracle's (which are
bitwise the reference's, test_oracle_golden.py); its transforms and F_E match
the reference-generated goldens; and the recorded T255 / T639 validation
against the reference itself (tests/golden/large_validation.npz)."""

import os

import numpy as np
import pytest

import swsdc_oracle as orc
import swsdc_stream as stm
from conftest import GOLDEN, TEST_PARAMS, rel_err


@pytest.mark.parametrize("R,I,J,bb", [(20, 64, 33, 1e5), (31, 96, 48, 2e5), (15, 48, 24, 1e12)])
def test_block_tables_bitwise_equal_dense(R, I, J, bb):
    d = orc.OraclePlan(R, I, J)
    st = stm.StreamPlan(R, I, J, bb)
    nblocks = 0
    for r0, r1, P, H in st.blocks(True):
        nblocks += 1
        assert np.array_equal(P, d.P[r0:r1, r0:])
        assert np.array_equal(H, d.H[r0:r1, r0:])
    assert nblocks == -(-(R + 1) // st.rb)


def test_stream_transforms_match_reference_goldens():
    g = np.load(os.path.join(GOLDEN, "transforms.npz"))
    for R, I, J in [(31, 96, 47), (31, 96, 48), (15, 48, 24), (63, 192, 96)]:
        tag = f"R{R}_I{I}_J{J}"
        st = stm.StreamPlan(R, I, J, block_bytes=2e5)   # several blocks
        assert rel_err(st.synthesize(g[f"{tag}_c"]), g[f"{tag}_syn"]) < 1e-14
        assert rel_err(st.analyze(g[f"{tag}_g"]), g[f"{tag}_ana"]) < 1e-14
        u, v = st.synth_uv(g[f"{tag}_c"], g[f"{tag}_c2"])
        assert rel_err(u, g[f"{tag}_u"]) < 1e-14 and rel_err(v, g[f"{tag}_v"]) < 1e-14
        d, c = st.anal_divcurl(g[f"{tag}_g"], g[f"{tag}_g2"])
        assert rel_err(d, g[f"{tag}_div"]) < 1e-14 and rel_err(c, g[f"{tag}_curl"]) < 1e-14


def test_stream_fe_matches_reference_goldens():
    g = np.load(os.path.join(GOLDEN, "rhs.npz"))
    prm = orc.OracleParams(**TEST_PARAMS)
    for R, I, J in [(15, 48, 24), (31, 96, 47), (31, 96, 48)]:
        tag = f"R{R}_I{I}_J{J}"
        st = stm.StreamPlan(R, I, J, block_bytes=1e5)
        for nl in (True, False):
            fe = stm.StreamRHS(st, prm, nl).eval_fe(g[f"{tag}_x"])
            want = g[f"{tag}_fe_nl{int(nl)}"]
            for f in range(3):
                if np.any(want[f] != 0):
                    assert rel_err(fe[f], want[f]) < 1e-13


def test_stream_mlsdc_step_matches_reference_golden():
    g = np.load(os.path.join(GOLDEN, "sweeps.npz"))
    prm = orc.OracleParams(**__import__("paper_1805_07923_b200.workloads", fromlist=["x"]).EARTH)
    h = orc.OracleHierarchy(stm.StreamLevel(31, 5, prm, (96, 48), block_bytes=1e5),
                            stm.StreamLevel(15, 3, prm, (48, 24), block_bytes=1e5))
    x = g["ml53_cs2_x"]
    ndf, ndc = orc.mlsdc_start(x, h)
    for _ in range(2):
        orc.mlsdc_iter(ndf, ndc, h, 240.0, 2)
    for f in range(3):
        assert rel_err(ndf.theta[-1][f], g["ml53_cs2_out"][f]) < 1e-12


def test_recorded_validation_against_reference():
    g = np.load(os.path.join(GOLDEN, "large_validation.npz"))
    for R in (255, 639):
        dev = g[f"dev_R{R}"]
        assert dev.shape == (10,)
        assert np.max(dev[:6]) <= 1e-14     # transforms
        assert np.max(dev[6:9]) <= 1e-13    # F_E
        assert dev[9] == 0.0                # one block: bitwise the reference
