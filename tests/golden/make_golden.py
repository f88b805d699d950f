"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `swsdc` from /root/reference/pkg/src (read-only), evaluates the
hot-path entry points on seeded inputs and writes compressed .npz fixtures
next to this file.  The fixtures are committed; nothing at test or bench
time reads /root/reference.  Inputs use the repo's seeded recipes
(paper_1805_07923_b200/workloads.py) and the reference test fixture recipe
(reference tests/conftest.py:20-39, restated below as `ref_random_*`).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from swsdc import mlsdc, sdc, spharm  # noqa: E402  (reference, read-only)
from swsdc.swe import ModelParams, PrognosticState, ShallowWaterRHS  # noqa: E402

from paper_1805_07923_b200 import workloads  # noqa: E402

TEST_PARAMS = dict(radius=6.37122e6, omega=7.292e-5, gravity=9.80616, nu=1.0e5, h_bar=29400.0)


def ref_random_coeffs(rng, R, scale=1.0, decay=0.15, zero_mean=False):
    c = np.zeros((R + 1, R + 1), dtype=complex)
    for r in range(R + 1):
        n = R + 1 - r
        env = scale * np.exp(-decay * np.arange(r, R + 1))
        c[r, r:] = (rng.normal(size=n) + 1j * rng.normal(size=n)) * env
    c[0] = c[0].real
    if zero_mean:
        c[0, 0] = 0.0
    return c


def ref_random_state(rng, R, phi_scale=300.0, wind_scale=1e-5):
    return np.stack([
        ref_random_coeffs(rng, R, phi_scale),
        ref_random_coeffs(rng, R, wind_scale, zero_mean=True),
        ref_random_coeffs(rng, R, wind_scale, zero_mean=True),
    ])


def to_ps(a):
    return PrognosticState(a[0].copy(), a[1].copy(), a[2].copy())


def from_ps(ps):
    return np.stack([ps.phi_prime, ps.zeta, ps.delta])


def plan_for(R, I, J):
    return spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)


def gen_grids():
    out = {}
    for n in (1, 2, 3, 7, 24, 47, 48, 96, 128, 191, 192, 384):
        mu, w = spharm.gauss_legendre_nodes(n)
        out[f"mu_{n}"] = mu
        out[f"w_{n}"] = w
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **out)


def gen_transforms():
    out = {}
    cases = [(31, 96, 47), (31, 96, 48), (15, 48, 24), (10, 33, 17), (63, 192, 96)]
    for R, I, J in cases:
        tag = f"R{R}_I{I}_J{J}"
        plan = plan_for(R, I, J)
        rng = np.random.default_rng(100 + R + J)
        c = ref_random_coeffs(rng, R)
        c2 = ref_random_coeffs(rng, R)
        g = rng.normal(size=(I, J))
        g2 = rng.normal(size=(I, J))
        out[f"{tag}_c"] = c
        out[f"{tag}_c2"] = c2
        out[f"{tag}_g"] = g
        out[f"{tag}_g2"] = g2
        out[f"{tag}_syn"] = plan.synthesize(c)
        out[f"{tag}_ana"] = plan.analyze(g)
        u, v = plan.synthesize_pair_cos_gradient(c, c2)
        out[f"{tag}_u"], out[f"{tag}_v"] = u, v
        d, k = plan.analyze_vector_div_curl(g, g2)
        out[f"{tag}_div"], out[f"{tag}_curl"] = d, k
        out[f"{tag}_fourier"] = plan._grid_to_fourier(g)
        if R <= 15:
            out[f"{tag}_P"] = plan._p
            out[f"{tag}_H"] = plan._h
    np.savez_compressed(os.path.join(HERE, "transforms.npz"), **out)


def gen_rhs():
    out = {}
    params = ModelParams(**TEST_PARAMS)
    for R, I, J in [(15, 48, 24), (31, 96, 47), (31, 96, 48)]:
        tag = f"R{R}_I{I}_J{J}"
        plan = plan_for(R, I, J)
        rng = np.random.default_rng(7 + R + J)
        x = ref_random_state(rng, R)
        out[f"{tag}_x"] = x
        for nl in (True, False):
            rhs = ShallowWaterRHS(plan, params, include_nonlinear=nl)
            out[f"{tag}_fe_nl{int(nl)}"] = from_ps(rhs.eval_f_e(to_ps(x)))
        rhs = ShallowWaterRHS(plan, params)
        out[f"{tag}_fi"] = from_ps(rhs.eval_f_i(to_ps(x)))
        for beta in (0.0, 112.5, 600.0):
            out[f"{tag}_solve_{beta}"] = from_ps(rhs.solve_implicit(to_ps(x), beta))
    np.savez_compressed(os.path.join(HERE, "rhs.npz"), **out)


def gen_sweeps():
    out = {}
    params = ModelParams(**workloads.EARTH)
    # single-level SDC: 3 and 5 nodes, T15 on its default grid
    for n_nodes, dt in ((3, 600.0), (5, 450.0)):
        lvl = mlsdc.build_level(15, n_nodes, params)
        x = workloads.seeded_state(15, 3)
        th = sdc.sdc_timestep(to_ps(x), dt, 2, lvl.tables, lvl.rhs)
        out[f"sdc{n_nodes}_x"] = x
        out[f"sdc{n_nodes}_out"] = from_ps(th)
    # MLSDC at small sizes: (3,2) one coarse sweep, (5,3) two coarse sweeps
    for (nf, nc, n_cs, Rf, Rc, gf, gc, dt) in (
        (3, 2, 1, 31, 15, (96, 48), (48, 24), 600.0),
        (5, 3, 2, 31, 15, (96, 48), (48, 24), 240.0),
    ):
        fine = mlsdc.build_level(Rf, nf, params, grid_shape=gf)
        coarse = mlsdc.build_level(Rc, nc, params, grid_shape=gc)
        ops = mlsdc.TransferOps.build(fine.tables.nodes, coarse.tables.nodes, Rf, Rc)
        hier = mlsdc.TwoLevelHierarchy(fine=fine, coarse=coarse, ops=ops)
        x = workloads.seeded_state(Rf, 5)
        sw_f, sw_c = mlsdc.initialize_mlsdc(to_ps(x), hier)
        for _ in range(2):
            if n_cs == 1:
                mlsdc.mlsdc_iteration(sw_f, sw_c, hier, dt)
            else:
                _iteration_multi_coarse(sw_f, sw_c, hier, dt, n_cs)
        tag = f"ml{nf}{nc}_cs{n_cs}"
        out[f"{tag}_x"] = x
        out[f"{tag}_out"] = from_ps(sw_f.theta[-1])
        out[f"{tag}_counts"] = np.array([
            fine.rhs.counters.solves, fine.rhs.counters.implicit_evals,
            fine.rhs.counters.explicit_evals, coarse.rhs.counters.solves,
            coarse.rhs.counters.implicit_evals, coarse.rhs.counters.explicit_evals])
    np.savez_compressed(os.path.join(HERE, "sweeps.npz"), **out)


def _iteration_multi_coarse(sw_fine, sw_coarse, hier, dt, n_cs):
    """mlsdc.mlsdc_iteration recomposed from the reference's public functions
    with n_cs coarse sweeps sharing one tau."""
    fine, coarse, ops = hier.fine, hier.coarse, hier.ops
    sdc.sdc_sweep(sw_fine, fine.tables, dt, fine.rhs)
    restricted = ops.restrict_states(sw_fine.theta)
    for m in range(1, coarse.n_nodes):
        sw_coarse.theta[m] = restricted[m]
        sw_coarse.f_i[m] = coarse.rhs.eval_f_i(restricted[m])
        sw_coarse.f_e[m] = coarse.rhs.eval_f_e(restricted[m])
    saved = [(t.copy(), a.copy(), b.copy()) for t, a, b in
             zip(sw_coarse.theta, sw_coarse.f_i, sw_coarse.f_e)]
    tau = mlsdc.compute_fas(sw_fine, sw_coarse, fine.tables, coarse.tables, dt, ops)
    for _ in range(n_cs):
        mlsdc.coarse_sweep_with_tau(sw_coarse, coarse.tables, dt, coarse.rhs, tau)
    n = coarse.n_nodes
    d_th = ops.interpolate_deltas([sw_coarse.theta[m] - saved[m][0] for m in range(n)])
    d_fi = ops.interpolate_deltas([sw_coarse.f_i[m] - saved[m][1] for m in range(n)])
    d_fe = ops.interpolate_deltas([sw_coarse.f_e[m] - saved[m][2] for m in range(n)])
    for m in range(1, sw_fine.n_nodes):
        sw_fine.theta[m] += d_th[m]
        sw_fine.f_i[m] += d_fi[m]
        sw_fine.f_e[m] += d_fe[m]


def gen_config0():
    """BASELINE config 0: T63 on 192x96 / T31 on 96x48, MLSDC(3,2,2), dt=600,
    one step from the seed-0 state."""
    params = ModelParams(**workloads.EARTH)
    fine = mlsdc.build_level(63, 3, params, grid_shape=(192, 96))
    coarse = mlsdc.build_level(31, 2, params, grid_shape=(96, 48))
    ops = mlsdc.TransferOps.build(fine.tables.nodes, coarse.tables.nodes, 63, 31)
    hier = mlsdc.TwoLevelHierarchy(fine=fine, coarse=coarse, ops=ops)
    x = workloads.seeded_state(63, 0)
    y = mlsdc.mlsdc_timestep(to_ps(x), 600.0, 2, hier)
    np.savez_compressed(os.path.join(HERE, "config0.npz"), x=x, out=from_ps(y))


from harness_runs import HARNESS_RUNS  # noqa: E402  (shared with tests/test_harness_host.py)


def gen_harness():
    """test-case initial states (reference testcases.py) and short
    run_simulation runs of every scheme with their cost counters, error norms
    and spectra (reference harness.py)."""
    from swsdc import harness, testcases  # reference, read-only
    out = {}
    R = 21
    n_lon, n_lat = spharm.default_grid_shape(R)
    plan = spharm.TransformPlan(spharm.build_gaussian_grid(n_lat, n_lon), R)
    for kind in testcases.CASE_KINDS:
        st, prm = testcases.build_initial_state(testcases.TestCaseSpec(kind), plan)
        out[f"init_{kind}"] = from_ps(st)
        out[f"init_{kind}_hbar"] = np.float64(prm.h_bar)
    states = {}
    for name, (case, scheme, rf, dt, t_end, it, nf, nc, alpha) in HARNESS_RUNS.items():
        cfg = harness.RunConfig(testcase=testcases.TestCaseSpec(case), scheme=scheme, r_fine=rf,
                                dt=dt, t_end=t_end, iterations=it, nodes_fine=nf,
                                nodes_coarse=nc, alpha=alpha)
        res = harness.run_simulation(cfg)
        states[name] = res.state
        out[f"run_{name}_state"] = from_ps(res.state)
        c = res.cost
        out[f"run_{name}_cost"] = np.array(
            [[x.solves, x.implicit_evals, x.explicit_evals]
             for x in (c.fine, c.coarse, c.fine_predicted, c.coarse_predicted, c.fine_init,
                       c.coarse_init)], dtype=np.int64)
        out[f"run_{name}_speedup"] = np.float64(c.theoretical_speedup or 0.0)
    rep = harness.compute_error_norms(states["sdc_dome"], states["irk2_rh"], plan)
    out["err_linf"] = np.array([rep.linf[v] for v in harness.STATE_VARS])
    out["err_l2"] = np.array([rep.l2[v] for v in harness.STATE_VARS])
    out["spectrum_zeta"] = harness.max_spectrum(states["mlsdc_jet"].zeta)
    np.savez_compressed(os.path.join(HERE, "harness.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "harness":
        gen_harness()
        sys.exit(0)
    gen_harness()
    gen_grids()
    gen_transforms()
    gen_rhs()
    gen_sweeps()
    gen_config0()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
