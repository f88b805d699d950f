"""GPU harness and test cases against the reference's own
results (tests/golden/harness.npz, tests/golden/make_golden.py):

* initial states of all four cases, analyzed on the GPU: <= 1e-11 relative;
* run_simulation for SDC, MLSDC(3,2), MLSDC(5,3) and IMEX-RK2: final state
  <= 1e-9 relative per field, cost counters (counted, predicted, init) exact;
* the CUDA-graph path equals the eager path (state to 1e-12, counters exact);
* compute_error_norms / max_spectrum on device results; the instability
  contract (reference tests/test_harness.py:213-224); determinism of CSVs."""

import dataclasses
import os
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu
sys.path.insert(0, GOLDEN)
from harness_runs import HARNESS_RUNS  # noqa: E402


@pytest.fixture(scope="module")
def hz():
    return np.load(os.path.join(GOLDEN, "harness.npz"))


def _cfg(name):
    from paper_1805_07923_b200 import harness
    from paper_1805_07923_b200.testcases import TestCaseSpec
    case, scheme, rf, dt, t_end, it, nf, nc, alpha = HARNESS_RUNS[name]
    return harness.RunConfig(testcase=TestCaseSpec(case), scheme=scheme, r_fine=rf, dt=dt,
                             t_end=t_end, iterations=it, nodes_fine=nf, nodes_coarse=nc,
                             alpha=alpha)


def _plan(R=21):
    from paper_1805_07923_b200 import spharm
    n_lon, n_lat = spharm.default_grid_shape(R)
    return spharm.TransformPlan(spharm.build_gaussian_grid(n_lat, n_lon), R)


def _fields_close(got, want, tol):
    """Per-field relative L-inf error; zeta and delta share one scale (the larger
    of the two), since a non-divergent case's delta is pure roundoff."""
    wind = max(np.max(np.abs(want[1])), np.max(np.abs(want[2])))
    for f in range(3):
        scale = np.max(np.abs(want[f])) if f == 0 else wind
        assert np.max(np.abs(got[f] - want[f])) / max(scale, 1e-300) < tol, f


@pytest.mark.parametrize("kind", ["steady_jet", "gaussian_dome", "rossby_haurwitz",
                                  "barotropic_instability"])
def test_initial_states_match_reference(hz, kind):
    from paper_1805_07923_b200 import testcases
    st, prm = testcases.build_initial_state(testcases.TestCaseSpec(kind), _plan())
    _fields_close(st.numpy(), hz[f"init_{kind}"], 1e-11)
    assert prm.h_bar == pytest.approx(float(hz[f"init_{kind}_hbar"]), rel=1e-13)


@pytest.mark.parametrize("name", list(HARNESS_RUNS))
def test_run_simulation_matches_reference(hz, name):
    from paper_1805_07923_b200 import harness
    res = harness.run_simulation(_cfg(name))
    _fields_close(res.state.numpy(), hz[f"run_{name}_state"], 1e-9)
    c = res.cost
    got = [[x.solves, x.implicit_evals, x.explicit_evals]
           for x in (c.fine, c.coarse, c.fine_predicted, c.coarse_predicted, c.fine_init,
                     c.coarse_init)]
    assert got == hz[f"run_{name}_cost"].tolist()
    assert c.matches_prediction()
    assert (c.theoretical_speedup or 0.0) == pytest.approx(float(hz[f"run_{name}_speedup"]),
                                                          rel=1e-14)


@pytest.mark.parametrize("name", ["sdc_dome", "mlsdc_jet"])
def test_graph_path_equals_eager(name):
    from paper_1805_07923_b200 import harness
    a = harness.run_simulation(_cfg(name))
    b = harness.run_simulation(_cfg(name), use_graph=True)
    assert rel_err(b.state.numpy(), a.state.numpy()) < 1e-12
    assert b.cost == a.cost


def test_error_norms_and_spectrum_match_reference(hz):
    from paper_1805_07923_b200 import harness
    plan = _plan()
    a = harness.run_simulation(_cfg("sdc_dome")).state
    b = harness.run_simulation(_cfg("irk2_rh")).state
    rep = harness.compute_error_norms(a, b, plan)
    for i, v in enumerate(harness.STATE_VARS):
        assert rep.linf[v] == pytest.approx(float(hz["err_linf"][i]), rel=1e-9)
        assert rep.l2[v] == pytest.approx(float(hz["err_l2"][i]), rel=1e-9)
    zero = harness.compute_error_norms(a, a, plan)
    assert all(zero.linf[v] == 0.0 and zero.l2[v] == 0.0 for v in harness.STATE_VARS)
    with pytest.raises(harness.UsageError):
        harness.compute_error_norms(a, a.truncated(10), plan)
    jet = harness.run_simulation(_cfg("mlsdc_jet")).state
    spec = harness.max_spectrum(jet.zeta)
    want = hz["spectrum_zeta"]
    assert np.max(np.abs(spec.cpu().numpy() - want)) / np.max(want) < 1e-9


def test_instability_reports_step_index():
    from paper_1805_07923_b200 import harness
    from paper_1805_07923_b200.testcases import TestCaseSpec
    cfg = harness.RunConfig(testcase=TestCaseSpec("gaussian_dome", nu=0.0), scheme="irk2",
                            r_fine=31, dt=30000.0, t_end=30000.0 * 40, iterations=1)
    with pytest.raises(harness.InstabilityError) as err:
        harness.run_simulation(cfg)
    assert 0 <= err.value.step < 40


def test_convergence_study_and_cost_csv(tmp_path):
    from paper_1805_07923_b200 import harness
    base = _cfg("sdc_dome")
    base = dataclasses.replace(base, nodes_fine=2, iterations=2)
    ref = dataclasses.replace(base, nodes_fine=5, iterations=8, dt=150.0)
    study = harness.convergence_study(base, [900.0, 600.0], ref)
    assert study.fit_slope("phi_prime", "linf") == pytest.approx(2.0, abs=0.5)
    with pytest.raises(harness.UsageError):
        harness.convergence_study(base, [600.0], dataclasses.replace(base, dt=600.0))
    res = harness.run_simulation(_cfg("mlsdc_jet"))
    p = tmp_path / "cost.csv"
    harness.write_cost_csv(res.cost, str(p))
    assert harness.read_cost_csv(str(p)) == res.cost
    # deterministic: identical runs give identical error CSVs
    texts = []
    for k in range(2):
        r = harness.run_simulation(_cfg("sdc_dome"))
        rep = harness.compute_error_norms(r.state, r.state * 0.0, r.plan, dt=600.0,
                                          scheme=r.config.label())
        q = tmp_path / f"e{k}.csv"
        harness.write_error_csv([rep], str(q))
        texts.append(q.read_text())
    assert texts[0] == texts[1]
