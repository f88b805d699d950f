"""Host-side logic of the harness / test-case drop-ins (no GPU): configuration
validation, labels, the cost model, speedups, slope fits and the CSV
contracts (reference tests/test_harness.py:49-75, 179-191, 238-287;
tests/test_testcases.py:31-37), with predicted counts pinned to the
reference's own runs (tests/golden/harness.npz)."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN  # noqa: E402


@pytest.fixture(scope="module")
def hz():
    return np.load(os.path.join(GOLDEN, "harness.npz"))


def _h():
    from paper_1805_07923_b200 import harness
    return harness


def _cfg(**kw):
    from paper_1805_07923_b200.testcases import TestCaseSpec
    base = dict(testcase=TestCaseSpec("gaussian_dome"), scheme="sdc", r_fine=31, dt=600.0,
                t_end=3600.0, iterations=4, nodes_fine=3)
    base.update(kw)
    return _h().RunConfig(**base)


def test_config_validation_and_labels():
    h = _h()
    with pytest.raises(h.UsageError):
        _cfg(scheme="rk4")
    with pytest.raises(h.UsageError):
        _cfg(dt=0.0)
    with pytest.raises(h.UsageError):
        _cfg(t_end=100.0)
    with pytest.raises(h.UsageError):
        _cfg(iterations=0)
    with pytest.raises(h.UsageError):
        _cfg(scheme="mlsdc", nodes_coarse=2)            # no r_coarse / alpha
    with pytest.raises(h.UsageError):
        _cfg(scheme="mlsdc", alpha=0.5)                 # no nodes_coarse
    with pytest.raises(h.UsageError):
        _cfg(t_end=1000.0).n_steps                     # not a multiple of dt
    c = _cfg(scheme="mlsdc", nodes_coarse=2, iterations=2, alpha=0.5)
    assert c.r_coarse == 16 and c.alpha == 16 / 31
    assert c.label() == "MLSDC(3,2,2,16/31)"
    assert _cfg().label() == "SDC(3,4)" and _cfg(scheme="irk2").label() == "IMEX-RK2"
    from paper_1805_07923_b200.testcases import TestCaseSpec
    with pytest.raises(ValueError):
        TestCaseSpec("tsunami")


def test_predicted_counts_match_reference_runs(hz):
    from paper_1805_07923_b200.testcases import TestCaseSpec
    h = _h()
    import sys
    sys.path.insert(0, GOLDEN)
    from harness_runs import HARNESS_RUNS
    for name, (case, scheme, rf, dt, t_end, it, nf, nc, alpha) in HARNESS_RUNS.items():
        cfg = h.RunConfig(testcase=TestCaseSpec(case), scheme=scheme, r_fine=rf, dt=dt,
                          t_end=t_end, iterations=it, nodes_fine=nf, nodes_coarse=nc, alpha=alpha)
        fp, cp = h.predicted_counts(cfg)
        want = hz[f"run_{name}_cost"]
        assert [fp.solves, fp.implicit_evals, fp.explicit_evals] == list(want[2]), name
        assert [cp.solves, cp.implicit_evals, cp.explicit_evals] == list(want[3]), name


def test_theoretical_and_observed_speedup():
    h = _h()
    assert h.theoretical_speedup(2, 1, 4, 2, 0.5, 256) == pytest.approx(1.66, abs=0.01)
    assert h.theoretical_speedup(4, 2, 8, 4, 0.5, 256) == pytest.approx(1.66, abs=0.01)
    assert h.theoretical_speedup(2, 2, 4, 2, 1.0, 256) == pytest.approx(0.75, abs=1e-12)
    with pytest.raises(h.UsageError):
        h.theoretical_speedup(2, 1, 4, 2, 1.5, 256)
    base = [(1e-2, 8.0), (1e-4, 32.0), (1e-6, 128.0)]
    fast = [(1e-2, 4.0), (1e-4, 16.0), (1e-6, 64.0)]
    assert h.observed_speedup(base, fast, 1e-3) == pytest.approx(2.0, rel=1e-12)


def test_slope_fit():
    h = _h()
    dts = [800.0, 400.0, 200.0, 100.0]
    ents = [h.StudyEntry(dt, True, h.ErrorReport(dt, "x", {"zeta": 3.0 * dt ** 4}, {"zeta": 1.0}))
            for dt in dts]
    st = h.StudyResult(ents, "ref", 50.0)
    assert st.fit_slope("zeta", "linf") == pytest.approx(4.0, abs=1e-9)
    with pytest.raises(h.UsageError):
        st.fit_slope("zeta", "linf", dts=[800.0])
    assert len(st.errors("zeta")) == 4


def test_csv_contracts(tmp_path):
    h = _h()
    from paper_1805_07923_b200.swe import EvalCounters
    rep = h.ErrorReport(dt=300.0, scheme="SDC(3,4)", linf={"phi_prime": 1.0, "zeta": 2.0, "delta": 3.0},
                        l2={"phi_prime": 0.1, "zeta": 0.2, "delta": 0.3}, wallclock_s=1.5)
    p = tmp_path / "errors.csv"
    h.write_error_csv([rep], str(p))
    lines = p.read_text(encoding="utf-8").splitlines()
    assert lines[0] == "dt,scheme,var,linf,l2,wallclock_s"
    assert lines[1].startswith("300,SDC(3,4),phi_prime,1,0.1") and len(lines) == 4
    p = tmp_path / "spectrum.csv"
    h.write_spectrum_csv(h.SpectrumReport("zeta", 0.0, np.array([0.5, 0.25, 0.0])), str(p))
    assert p.read_text(encoding="utf-8").splitlines() == ["n0,max_abs", "0,0.5", "1,0.25", "2,0"]
    cost = h.CostReport("MLSDC(3,2,2,16/31)", 6, EvalCounters(12, 12, 12), EvalCounters(6, 12, 12),
                        EvalCounters(12, 12, 12), EvalCounters(6, 12, 12), EvalCounters(0, 6, 6),
                        EvalCounters(0, 6, 6), 1.6603)
    p = tmp_path / "cost.csv"
    h.write_cost_csv(cost, str(p))
    assert h.read_cost_csv(str(p)) == cost
    (tmp_path / "bad.csv").write_text("a,b\n")
    with pytest.raises(h.UsageError):
        h.read_cost_csv(str(tmp_path / "bad.csv"))


def test_jet_profile_and_phase_speed():
    from paper_1805_07923_b200 import testcases as tc
    phi = np.linspace(-math.pi / 2, math.pi / 2, 1001)
    u = tc.jet_profile(phi, 80.0, math.pi / 7, math.pi / 2 - math.pi / 7)
    assert np.all(u[(phi <= math.pi / 7) | (phi >= math.pi / 2 - math.pi / 7)] == 0.0)
    assert u.max() == pytest.approx(80.0, rel=1e-3)
    c = tc.haurwitz_phase_speed()
    assert c == pytest.approx((4 * 7 * 7.848e-6 - 2 * 7.292e-5) / 30.0, rel=1e-15)
