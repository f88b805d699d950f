"""Edge cases of the GPU path against the CPU oracle: the smallest truncations
(default dealiased grids, n_lon from 1 to 64: every FFT path, odd J with an
equator pair), batch sizes around the internal grouping (16 vectors per
analysis group, 4-6 fields per synthesis CTA), ensembles of F_E, non-contiguous
inputs, and the reference's usage/numerical error contract
(reference spharm.py:192-195, implicit.py:31-49, swe.py:56-58)."""

import numpy as np
import pytest
import torch

from conftest import TEST_PARAMS, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _rand_coeffs(rng, R, n=None):
    shape = (R + 1, R + 1) if n is None else (n, R + 1, R + 1)
    c = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    c = np.triu(c)
    c[..., 0, :] = c[..., 0, :].real
    return c


def _plans(R):
    import swsdc_oracle as orc
    from paper_1805_07923_b200 import spharm
    n_lon, n_lat = spharm.default_grid_shape(R)
    return (spharm.TransformPlan(spharm.build_gaussian_grid(n_lat, n_lon), R),
            orc.OraclePlan(R, n_lon, n_lat))


@pytest.mark.parametrize("R", [0, 1, 2, 3, 4, 5, 7, 10, 21])
def test_small_truncations_match_oracle(R):
    rng = np.random.default_rng(R)
    plan, oplan = _plans(R)
    c = _rand_coeffs(rng, R)
    g = plan.synthesize(c)
    assert rel_err(g, oplan.synthesize(c)) < TOL
    g2 = rng.normal(size=g.shape)
    assert rel_err(plan.analyze(g2), oplan.analyze(g2)) < TOL
    if R >= 1:
        psi, chi = _rand_coeffs(rng, R), _rand_coeffs(rng, R)
        u, v = plan.synthesize_pair_cos_gradient(psi, chi)
        uo, vo = oplan.synth_uv(psi, chi)
        assert rel_err(u, uo) < TOL and rel_err(v, vo) < TOL
        gv = rng.normal(size=g.shape)
        d, k = plan.analyze_vector_div_curl(g2, gv)
        do, ko = oplan.anal_divcurl(g2, gv)
        assert rel_err(d, do) < TOL and rel_err(k, ko) < TOL


@pytest.mark.parametrize("R", [1, 3, 5, 10, 21])
@pytest.mark.parametrize("nl", [True, False])
def test_small_truncation_eval_fe_matches_oracle(R, nl):
    import swsdc_oracle as orc
    from paper_1805_07923_b200 import swe
    rng = np.random.default_rng(100 + R)
    plan, oplan = _plans(R)
    x = np.stack([_rand_coeffs(rng, R) * s for s in (1e3, 1e-5, 1e-6)])
    rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**TEST_PARAMS), include_nonlinear=nl)
    orhs = orc.OracleRHS(oplan, orc.OracleParams(**TEST_PARAMS), nl)
    got = rhs.eval_f_e(swe.PrognosticState(torch.as_tensor(x).cuda())).numpy()
    want = orhs.eval_fe(x)
    for f in range(3):
        assert rel_err(got[f], want[f]) < 1e-10, f


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 7, 16, 17, 31, 33])
def test_batch_sizes_match_oracle(batch):
    rng = np.random.default_rng(batch)
    R = 21
    plan, oplan = _plans(R)
    c = _rand_coeffs(rng, R, batch)
    g = plan.synthesize(torch.as_tensor(c).cuda()).cpu().numpy()
    want = np.stack([oplan.synthesize(ci) for ci in c])
    assert rel_err(g, want) < TOL
    back = plan.analyze(torch.as_tensor(want).cuda()).cpu().numpy()
    assert rel_err(back, np.stack([oplan.analyze(gi) for gi in want])) < TOL


@pytest.mark.parametrize("members", [2, 4, 5, 17, 64])
def test_batched_eval_fe_equals_per_member(members):
    """Even member counts take the member-pair analysis (two members per CTA
    sharing the q tiles), odd ones the per-member kernel."""
    from paper_1805_07923_b200 import swe
    rng = np.random.default_rng(members)
    R = 21
    plan, _ = _plans(R)
    x = np.stack([np.stack([_rand_coeffs(rng, R) * s for s in (1e3, 1e-5, 1e-6)])
                  for _ in range(members)])
    rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**TEST_PARAMS))
    batched = rhs.eval_f_e(swe.PrognosticState(torch.as_tensor(x).cuda())).numpy()
    for m in range(members):
        single = rhs.eval_f_e(swe.PrognosticState(torch.as_tensor(x[m]).cuda())).numpy()
        # the batch size may select another grid-stage path or latitude split
        # (different summation order), so equal to rounding, not bitwise
        for f in range(3):
            assert rel_err(batched[m][f], single[f]) < 1e-12, (m, f)


def test_non_contiguous_and_numpy_inputs():
    rng = np.random.default_rng(7)
    R = 10
    plan, oplan = _plans(R)
    c = _rand_coeffs(rng, R, 4)
    t = torch.as_tensor(np.ascontiguousarray(c.transpose(1, 2, 0))).cuda().permute(2, 0, 1)
    assert not t.is_contiguous()
    got = plan.synthesize(t).cpu().numpy()
    assert rel_err(got, np.stack([oplan.synthesize(ci) for ci in c])) < TOL
    host = plan.synthesize(c)                   # numpy in -> numpy out
    assert isinstance(host, np.ndarray) and rel_err(host, got) < 1e-15


def test_usage_and_numerical_errors():
    from paper_1805_07923_b200 import implicit, spharm, swe
    R = 10
    plan, _ = _plans(R)
    with pytest.raises(ValueError):
        spharm.TransformPlan(spharm.build_gaussian_grid(8, 16), 10)        # n_lon < 2R+1
    with pytest.raises(ValueError):
        plan.synthesize(np.zeros((R + 2, R + 2), complex))                 # R_in > R
    with pytest.raises(ValueError):
        plan.analyze(np.zeros((plan.grid.n_lon + 1, plan.grid.n_lat)))      # wrong grid
    with pytest.raises(ValueError):
        swe.PrognosticState(np.zeros((R + 1, R + 1), complex), np.zeros((R, R), complex),
                            np.zeros((R + 1, R + 1), complex))
    rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**TEST_PARAMS))
    st = swe.PrognosticState(torch.zeros((3, R + 1, R + 1), dtype=torch.complex128).cuda())
    with pytest.raises(ValueError):
        rhs.solve_implicit(st, -1.0)                                        # beta < 0
    with pytest.raises(ValueError):
        swe.ModelParams(**{**TEST_PARAMS, "h_bar": -1.0})                  # non-physical depth


def test_spec_combine_multi_equals_single_launches():
    """The batched restriction/FAS/interpolation launches give bitwise the same
    sums as one spec_combine per output (same terms, same order), including
    in-place outputs and mixed input truncations."""
    from paper_1805_07923_b200 import swe
    rng = np.random.default_rng(3)
    dev = torch.device("cuda")
    xs = [torch.as_tensor(_rand_coeffs(rng, R, 3), device=dev) for R in (21, 10, 21, 15)]
    jobs = [([1.0, -0.5, 0.25], [xs[0], xs[1], xs[3]], None),
            ([2.0, 1.0], [xs[3], xs[2]], None),
            ([1.0, 0.5, -0.5], [xs[2].clone(), xs[0], xs[1]], None)]
    jobs[2] = (jobs[2][0], jobs[2][1], jobs[2][1][0])          # in place on its own input
    want = [swe.spec_combine(w, [t.clone() for t in x], 21) for w, x, _ in jobs]
    got = swe.spec_combine_multi(jobs, 21)
    for g, w in zip(got, want):
        assert torch.equal(g, w)
    many = [([1.0, 1.0], [xs[0], xs[2]], None) for _ in range(40)]   # > 16 outputs: chunked
    outs = swe.spec_combine_multi(many, 15)
    ref = swe.spec_combine([1.0, 1.0], [xs[0], xs[2]], 15)
    assert all(torch.equal(o, ref) for o in outs)


@pytest.mark.parametrize("batch", [2, 3, 6])
def test_batched_div_curl_equals_per_member(batch):
    """analyze_vector_div_curl over a batch (4 analysis vectors per member: the
    member-pair path for even batches) equals the per-member calls."""
    rng = np.random.default_rng(100 + batch)
    R = 31
    plan, _ = _plans(R)
    c = _rand_coeffs(rng, R, 2 * batch)
    u = plan.synthesize(torch.as_tensor(c[:batch]).cuda())
    v = plan.synthesize(torch.as_tensor(c[batch:]).cuda())
    d, k = plan.analyze_vector_div_curl(u, v)
    for b in range(batch):
        d1, k1 = plan.analyze_vector_div_curl(u[b], v[b])
        assert rel_err(d[b].cpu().numpy(), d1.cpu().numpy()) < 1e-12
        assert rel_err(k[b].cpu().numpy(), k1.cpu().numpy()) < 1e-12
