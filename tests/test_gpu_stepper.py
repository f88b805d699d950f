"""CUDA-graph steppers (paper_1805_07923_b200/stepper.py) vs reference goldens
and the oracle: config 0 step, multi-step trajectories, ensembles, counters."""

import os

import numpy as np
import pytest
import torch

import swsdc_oracle as orc
from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu


def earth():
    from paper_1805_07923_b200 import swe, workloads
    return swe.ModelParams(**workloads.EARTH), orc.OracleParams(**workloads.EARTH)


def test_graph_stepper_config0_matches_reference():
    from paper_1805_07923_b200 import mlsdc, stepper, swe
    g = np.load(os.path.join(GOLDEN, "config0.npz"))
    params, _ = earth()
    hier = mlsdc.build_hierarchy(params, 63, 3, 31, 2, grid_fine=(192, 96), grid_coarse=(96, 48))
    st = stepper.MLSDCStepper(hier, 600.0, 2, swe.PrognosticState(torch.as_tensor(g["x"]).cuda()))
    y = st.run(1).numpy()
    for f in range(3):
        assert rel_err(y[f], g["out"][f]) < 1e-9
    # counters: init 1+1, per iteration M_f fine and 2 M_c coarse evaluations (harness.py:125-143)
    fc, cc = st.counts_per_step
    assert (fc.solves, fc.implicit_evals, fc.explicit_evals) == (4, 5, 5)
    assert (cc.solves, cc.implicit_evals, cc.explicit_evals) == (2, 5, 5)


def test_graph_stepper_trajectory_and_ensemble_match_oracle():
    from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads
    params, oparams = earth()
    hier = mlsdc.build_hierarchy(params, 31, 5, 15, 3, grid_fine=(96, 48), grid_coarse=(48, 24))
    x = np.stack([workloads.seeded_state(31, k) for k in range(3)])
    st = stepper.MLSDCStepper(hier, 240.0, 2, swe.PrognosticState(torch.as_tensor(x).cuda()),
                              n_coarse_sweeps=2)
    y = st.run(3).numpy()
    oh = orc.OracleHierarchy(orc.OracleLevel(31, 5, oparams, (96, 48)),
                             orc.OracleLevel(15, 3, oparams, (48, 24)))
    for m in range(3):
        want = x[m]
        for _ in range(3):
            want = orc.mlsdc_step(want, 240.0, 2, oh, coarse_sweeps=2)
        for f in range(3):
            assert rel_err(y[m, f], want[f]) < 1e-9


def test_sdc_stepper_matches_oracle():
    from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads
    params, oparams = earth()
    lvl = mlsdc.build_level(15, 3, params)
    x = workloads.seeded_state(15, 4)
    st = stepper.SDCStepper(lvl, 600.0, 3, swe.PrognosticState(torch.as_tensor(x).cuda()))
    y = st.run(2).numpy()
    ol = orc.OracleLevel(15, 3, oparams)
    want = orc.sdc_step(orc.sdc_step(x, 600.0, 3, ol.tb, ol.rhs), 600.0, 3, ol.tb, ol.rhs)
    for f in range(3):
        assert rel_err(y[f], want[f]) < 1e-9


def test_instability_is_reported_with_step_index():
    from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads
    params, _ = earth()
    hier = mlsdc.build_hierarchy(params, 15, 3, 7, 2)
    x = workloads.seeded_state(15, 0) * 1e30  # blows up
    st = stepper.MLSDCStepper(hier, 3600.0, 2, swe.PrognosticState(torch.as_tensor(x).cuda()))
    with pytest.raises(stepper.InstabilityError) as ei:
        st.run(50)
    assert 0 <= ei.value.step < 50   # 0-based, as the reference loop index


def test_eager_growth_after_capture_keeps_the_graph_valid():
    """A captured step bakes the plan workspaces into its graph; an eager call
    on the same plan that needs more scratch (a bigger batch) must not free
    them (capi.cu ensure_ws / grow_grid_ws retire pinned buffers)."""
    from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads
    params, oparams = earth()
    hier = mlsdc.build_hierarchy(params, 31, 3, 15, 2, grid_fine=(96, 48), grid_coarse=(48, 24))
    x = workloads.seeded_state(31, 6)
    st = stepper.MLSDCStepper(hier, 600.0, 2, swe.PrognosticState(torch.as_tensor(x).cuda()))
    st.run(1)
    # eager F_E and analyses on a much larger batch through the same plans
    big = torch.as_tensor(np.stack([workloads.seeded_state(31, k) for k in range(40)])).cuda()
    hier.fine.rhs.eval_f_e(swe.PrognosticState(big))
    grids = hier.fine.plan.synthesize(big.reshape(-1, 32, 32))
    hier.fine.plan.analyze(grids)
    torch.cuda.synchronize()
    st.set_state(swe.PrognosticState(torch.as_tensor(x).cuda()))
    y = st.run(1).numpy()
    oh = orc.OracleHierarchy(orc.OracleLevel(31, 3, oparams, (96, 48)),
                             orc.OracleLevel(15, 2, oparams, (48, 24)))
    want = orc.mlsdc_step(x, 600.0, 2, oh)
    for f in range(3):
        assert rel_err(y[f], want[f]) < 1e-9
