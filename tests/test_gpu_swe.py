"""GPU shallow-water operators vs reference golden vectors."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, TEST_PARAMS, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "rhs.npz"))


def rhs_for(R, I, J, nl=True):
    from paper_1805_07923_b200 import spharm, swe
    plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
    return swe.ShallowWaterRHS(plan, swe.ModelParams(**TEST_PARAMS), include_nonlinear=nl)


CASES = [(15, 48, 24), (31, 96, 47), (31, 96, 48)]


@pytest.mark.parametrize("R,I,J", CASES)
@pytest.mark.parametrize("nl", [True, False])
def test_eval_f_e_matches_reference(golden, R, I, J, nl):
    from paper_1805_07923_b200 import swe
    tag = f"R{R}_I{I}_J{J}"
    rhs = rhs_for(R, I, J, nl)
    got = rhs.eval_f_e(swe.PrognosticState(golden[f"{tag}_x"])).numpy()
    want = golden[f"{tag}_fe_nl{int(nl)}"]
    for f in range(3):
        assert rel_err(got[f], want[f]) < 1e-11, f
    assert rhs.counters.explicit_evals == 1


@pytest.mark.parametrize("R,I,J", CASES)
def test_eval_f_i_and_solve_match_reference(golden, R, I, J):
    from paper_1805_07923_b200 import swe
    tag = f"R{R}_I{I}_J{J}"
    rhs = rhs_for(R, I, J)
    x = swe.PrognosticState(golden[f"{tag}_x"])
    assert rel_err(rhs.eval_f_i(x).numpy(), golden[f"{tag}_fi"]) < 1e-14
    for beta in (0.0, 112.5, 600.0):
        got = rhs.solve_implicit(x, beta).numpy()
        for f in range(3):
            assert rel_err(got[f], golden[f"{tag}_solve_{beta}"][f]) < 1e-13
    assert rhs.counters.solves == 3 and rhs.counters.implicit_evals == 1
