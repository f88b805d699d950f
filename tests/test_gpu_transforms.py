"""GPU transforms vs golden vectors from the reference (tests/golden/make_golden.py)
and vs the CPU oracle.  Tolerance: 1e-11 relative L-inf per transform
(BASELINE.json north_star)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "transforms.npz"))


def plan_for(R, I, J):
    from paper_1805_07923_b200 import spharm
    return spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)


CASES = [(31, 96, 47), (31, 96, 48), (15, 48, 24), (10, 33, 17), (63, 192, 96)]


@pytest.mark.parametrize("R,I,J", CASES)
def test_synthesize_matches_reference(golden, R, I, J):
    tag = f"R{R}_I{I}_J{J}"
    plan = plan_for(R, I, J)
    got = plan.synthesize(golden[f"{tag}_c"])
    assert rel_err(got, golden[f"{tag}_syn"]) < TOL


@pytest.mark.parametrize("R,I,J", CASES)
def test_analyze_matches_reference(golden, R, I, J):
    tag = f"R{R}_I{I}_J{J}"
    plan = plan_for(R, I, J)
    got = plan.analyze(golden[f"{tag}_g"])
    assert rel_err(got, golden[f"{tag}_ana"]) < TOL


@pytest.mark.parametrize("R,I,J", CASES)
def test_vector_transforms_match_reference(golden, R, I, J):
    tag = f"R{R}_I{I}_J{J}"
    plan = plan_for(R, I, J)
    u, v = plan.synthesize_pair_cos_gradient(golden[f"{tag}_c"], golden[f"{tag}_c2"])
    assert rel_err(u, golden[f"{tag}_u"]) < TOL
    assert rel_err(v, golden[f"{tag}_v"]) < TOL
    d, k = plan.analyze_vector_div_curl(golden[f"{tag}_g"], golden[f"{tag}_g2"])
    assert rel_err(d, golden[f"{tag}_div"]) < TOL
    assert rel_err(k, golden[f"{tag}_curl"]) < TOL


def test_batched_transforms_match_oracle():
    import swsdc_oracle as orc
    from paper_1805_07923_b200 import workloads
    R, I, J = 63, 192, 96
    plan = plan_for(R, I, J)
    oplan = orc.OraclePlan(R, I, J)
    c = workloads.transform_batch(R, 15)
    g = plan.synthesize(torch.as_tensor(c).cuda())
    want = np.stack([oplan.synthesize(ci) for ci in c])
    assert rel_err(g.cpu().numpy(), want) < TOL
    back = plan.analyze(g)
    want_b = np.stack([oplan.analyze(gi) for gi in want])
    assert rel_err(back.cpu().numpy(), want_b) < TOL
    assert rel_err(back.cpu().numpy(), c) < TOL


def test_pinned_host_upload_and_download(golden):
    """synthesize() of a pinned host tensor uploads only the s >= r triangle (the
    lower triangle, garbage here, must not be read) and analyze(out=pinned host)
    copies the result back; both equal the device-resident path bit for bit."""
    from paper_1805_07923_b200 import spharm
    R, I, J = 31, 96, 48
    plan = plan_for(R, I, J)
    c = np.stack([golden[f"R{R}_I{I}_J{J}_c"]] * 3)
    dirty = c.copy()
    lo = np.tril_indices(R + 1, -1)
    dirty[:, lo[0], lo[1]] = 1e300 + 7j
    host = torch.from_numpy(dirty).pin_memory()
    dev = spharm.upload_coeffs(host)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), c)
    g_ref = plan.synthesize(torch.from_numpy(c).cuda())
    g_host = plan.synthesize(host)
    assert g_host.is_cuda and torch.equal(g_ref, g_host)
    o_pin = torch.empty(c.shape, dtype=torch.complex128).pin_memory()
    assert plan.analyze(g_ref, out=o_pin) is o_pin
    torch.cuda.synchronize()
    assert torch.equal(o_pin, plan.analyze(g_ref).cpu())
    sentinel = torch.full(c.shape, 3 + 4j, dtype=torch.complex128).pin_memory()
    spharm.download_coeffs(dev, sentinel, write_lower=False)
    dense = torch.full(c.shape, 3 + 4j, dtype=torch.complex128).pin_memory()
    spharm.download_coeffs(dev, dense)
    torch.cuda.synchronize()
    assert np.array_equal(dense.numpy(), c)
    tri = np.triu_indices(R + 1)
    assert np.array_equal(sentinel.numpy()[:, tri[0], tri[1]], c[:, tri[0], tri[1]])
    below = sentinel.numpy()[:, lo[0], lo[1]]
    assert np.all((below == 3 + 4j) | (below == 0))      # untouched, or the device's zeros
    assert np.mean(below == 3 + 4j) > 0.5                # ... and mostly not sent at all
    with pytest.raises(ValueError):
        spharm.upload_coeffs(torch.from_numpy(c))          # pageable: refused
    with pytest.raises(ValueError):
        plan.analyze(g_ref, out=torch.empty(c.shape, dtype=torch.complex128))


def test_tma_and_forced_split_variants_match_reference(tmp_path):
    """The opt-in TMA analysis (SWSDC_ANA_TMA=2), the DFMA analysis kept for the
    DMMA-vs-DFMA comparison (SWSDC_ANA_DFMA=1), every forced latitude split
    (SWSDC_ANA_LSPLIT=1..4) and the unspecialised last chunk give the reference's
    analysis; the knobs are read once per process, so each runs in a subprocess."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "from conftest import GOLDEN, rel_err;"
        "from paper_1805_07923_b200 import spharm;"
        "g = np.load(GOLDEN + '/transforms.npz');"
        "worst = 0.0\n"
        "for R, I, J in [(31, 96, 48), (63, 192, 96), (31, 96, 47)]:\n"
        "    t = f'R{R}_I{I}_J{J}'\n"
        "    plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)\n"
        "    for nb in (1, 7, 16):\n"
        "        f = np.stack([g[t + '_g']] * nb)\n"
        "        worst = max(worst, rel_err(plan.analyze(f)[0], g[t + '_ana']))\n"
        "print(worst)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"SWSDC_ANA_TMA": "2"}, {"SWSDC_ANA_LSPLIT": "1"}, {"SWSDC_ANA_LSPLIT": "2"},
                {"SWSDC_ANA_LSPLIT": "3"}, {"SWSDC_ANA_LSPLIT": "4"}, {"SWSDC_ANA_DFMA": "1"},
                {"SWSDC_ANA_DFMA": "1", "SWSDC_ANA_LSPLIT": "3"}, {"SWSDC_ANA_SHORT": "0"}):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True,
                             text=True, env={**os.environ, **env}, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        assert float(out.stdout.strip().splitlines()[-1]) < TOL, (env, out.stdout)


def test_packed_upload_matches_host():
    """SWSDC_UPLOAD_MODE=2 (host-packed triangles, stream gated by a stream memory
    operation, one contiguous copy, device expansion): more batches than staging
    slots, of changing size (slot reallocation), on two streams, each equal to the
    host matrices with a zero lower triangle; small transfers keep the zero-copy
    kernel.  The knob is read once per process, hence the subprocess."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, '.');"
        "from paper_1805_07923_b200 import spharm, _lib;"
        "rng = np.random.default_rng(5); bad = 0\n"
        "streams = [torch.cuda.Stream(), torch.cuda.Stream()]\n"
        "n0 = _lib.launch_count()\n"
        "jobs = []\n"
        "for k, (R, nm) in enumerate([(255, 15), (255, 15), (127, 40), (255, 3), (255, 15), (170, 9),"
        " (255, 15), (255, 15), (255, 15), (255, 30), (255, 15), (31, 2)]):\n"
        "    c = rng.standard_normal((nm, R + 1, R + 1)) + 1j * rng.standard_normal((nm, R + 1, R + 1))\n"
        "    host = torch.from_numpy(c).pin_memory()\n"
        "    with torch.cuda.stream(streams[k % 2]):\n"
        "        dev = spharm.upload_coeffs(host)\n"
        "    jobs.append((c, host, dev))\n"
        "torch.cuda.synchronize()\n"
        "for c, host, dev in jobs:\n"
        "    bad += not np.array_equal(dev.cpu().numpy(), np.triu(c))\n"
        "print(bad)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"SWSDC_UPLOAD_MODE": "2"}, {"SWSDC_UPLOAD_MODE": "2", "SWSDC_PACK_THREADS": "3"},
                {"SWSDC_UPLOAD_MODE": "0"}, {"SWSDC_UPLOAD_MODE": "1"}):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True,
                             text=True, env={**os.environ, **env}, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        assert int(out.stdout.strip().splitlines()[-1]) == 0, (env, out.stdout)


@pytest.mark.parametrize("R,I,J", [(63, 1920, 96), (31, 3840, 48), (47, 1920, 73)])
def test_long_rings_match_oracle(R, I, J):
    """n_lon = 15 * 32 K rings (T639 / T1279 grids: one latitude pair per CTA)
    take the ring_fft15 kernels (15-point prime-factor DFT + register FFTs of
    32 K points) in synthesize / analyze / div-curl and in the split F_E path;
    small truncations keep the numpy oracle cheap."""
    import swsdc_oracle as orc
    from paper_1805_07923_b200 import spharm, swe, workloads
    plan = plan_for(R, I, J)
    oplan = orc.OraclePlan(R, I, J)
    c = workloads.transform_batch(R, 3)
    g = plan.synthesize(torch.as_tensor(c).cuda()).cpu().numpy()
    want = np.stack([oplan.synthesize(ci) for ci in c])
    assert rel_err(g, want) < TOL
    back = plan.analyze(torch.as_tensor(want).cuda()).cpu().numpy()
    assert rel_err(back, np.stack([oplan.analyze(gi) for gi in want])) < TOL
    u, v = plan.synthesize_pair_cos_gradient(c[0], c[1])
    ou, ov = oplan.synth_uv(c[0], c[1])
    assert rel_err(u, ou) < TOL and rel_err(v, ov) < TOL
    d, k = plan.analyze_vector_div_curl(want[0], want[1])
    od, ok = oplan.anal_divcurl(want[0], want[1])
    assert rel_err(d, od) < TOL and rel_err(k, ok) < TOL
    params = swe.ModelParams(**workloads.EARTH)
    orhs = orc.OracleRHS(oplan, orc.OracleParams(**workloads.EARTH))
    x = workloads.seeded_state(R, 3)
    fe = swe.ShallowWaterRHS(plan, params).eval_f_e(
        swe.PrognosticState(torch.as_tensor(x).cuda())).numpy()
    ofe = orhs.eval_fe(x)
    for f in range(3):
        assert rel_err(fe[f], ofe[f]) < TOL


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24])
@pytest.mark.parametrize("members", [1, 3])
def test_every_register_fft_length_matches_oracle(K, members):
    """Every ring length with a register FFT (n_lon = 32 K): the half-exchange
    shuffle stages (even K) and the full-exchange ones (odd K), decimation in
    frequency (f2g / g2f, the fused kernel's inverse transforms) and in time (its
    forward transforms), at truncations that fill the band (3/2 rule) on a few
    latitudes, single states and ensembles -- against the numpy oracle."""
    import swsdc_oracle as orc
    from paper_1805_07923_b200 import spharm, swe, workloads
    I = 32 * K
    R = max(1, min((I - 1) // 3, 42))
    J = 10
    plan = plan_for(R, I, J)
    oplan = orc.OraclePlan(R, I, J)
    c = workloads.transform_batch(R, 2)
    g = plan.synthesize(torch.as_tensor(c).cuda()).cpu().numpy()
    want = np.stack([oplan.synthesize(ci) for ci in c])
    assert rel_err(g, want) < TOL
    back = plan.analyze(torch.as_tensor(want).cuda()).cpu().numpy()
    assert rel_err(back, np.stack([oplan.analyze(gi) for gi in want])) < TOL
    params = swe.ModelParams(**workloads.EARTH)
    orhs = orc.OracleRHS(oplan, orc.OracleParams(**workloads.EARTH))
    x = np.stack([workloads.seeded_state(R, k) for k in range(members)])
    fe = swe.ShallowWaterRHS(plan, params).eval_f_e(
        swe.PrognosticState(torch.as_tensor(x if members > 1 else x[0]).cuda())).numpy()
    fe = fe if members > 1 else fe[None]
    for m in range(members):
        ofe = orhs.eval_fe(x[m])
        for f in range(3):
            assert rel_err(fe[m][f], ofe[f]) < TOL, (m, f)


def test_round2_kernel_variants_match_reference():
    """Round-2 alternatives behind knobs (read once per process, so each runs in a
    subprocess): the opt-in tensor-core synthesis (SWSDC_SYN_DMMA=1, 4/8/16 fields
    per CTA), the recurrence-only analysis (SWSDC_TABLES=0), the 12-FFT fused grid
    kernel (SWSDC_SWE_G5=0) and the column-major F_E layout (SWSDC_FE_PM=0) give
    the reference's synthesis and F_E."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "from conftest import GOLDEN, TEST_PARAMS, rel_err;"
        "from paper_1805_07923_b200 import spharm, swe;"
        "g = np.load(GOLDEN + '/transforms.npz'); h = np.load(GOLDEN + '/rhs.npz');"
        "worst = 0.0\n"
        "for R, I, J in [(31, 96, 48), (63, 192, 96), (31, 96, 47)]:\n"
        "    t = f'R{R}_I{I}_J{J}'\n"
        "    plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)\n"
        "    for nb in (3, 8, 15, 20):\n"
        "        c = np.stack([g[t + '_c']] * nb)\n"
        "        s = plan.synthesize(c)\n"
        "        worst = max(worst, max(rel_err(s[k], g[t + '_syn']) for k in range(nb)))\n"
        "for R, I, J in [(15, 48, 24), (31, 96, 47), (31, 96, 48)]:\n"
        "    t = f'R{R}_I{I}_J{J}'\n"
        "    plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)\n"
        "    rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**TEST_PARAMS))\n"
        "    fe = rhs.eval_f_e(swe.PrognosticState(h[t + '_x'])).numpy()\n"
        "    worst = max(worst, max(rel_err(fe[f], h[t + '_fe_nl1'][f]) for f in range(3)))\n"
        "print(worst)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"SWSDC_SYN_DMMA": "1"}, {"SWSDC_SYN_DMMA": "1", "SWSDC_SYN_DMMA_GF": "4"},
                {"SWSDC_SYN_DMMA": "1", "SWSDC_SYN_DMMA_GF": "16"}, {"SWSDC_TABLES": "0"},
                {"SWSDC_SWE_G5": "0"}, {"SWSDC_FE_PM": "0"}):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True,
                             text=True, env={**os.environ, **env}, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        assert float(out.stdout.strip().splitlines()[-1]) < TOL, (env, out.stdout)
