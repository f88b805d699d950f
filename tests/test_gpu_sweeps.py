"""GPU SDC / MLSDC steps vs reference golden vectors (1e-9 per step)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "sweeps.npz"))


def test_sdc_timesteps_match_reference(golden):
    from paper_1805_07923_b200 import mlsdc, sdc, swe, workloads
    params = swe.ModelParams(**workloads.EARTH)
    for n_nodes, dt in ((3, 600.0), (5, 450.0)):
        lvl = mlsdc.build_level(15, n_nodes, params)
        x = swe.PrognosticState(golden[f"sdc{n_nodes}_x"])
        y = sdc.sdc_timestep(x, dt, 2, lvl.tables, lvl.rhs).numpy()
        want = golden[f"sdc{n_nodes}_out"]
        for f in range(3):
            assert rel_err(y[f], want[f]) < 1e-9


@pytest.mark.parametrize("nf,nc,ncs,dt", [(3, 2, 1, 600.0), (5, 3, 2, 240.0)])
def test_mlsdc_matches_reference(golden, nf, nc, ncs, dt):
    from paper_1805_07923_b200 import mlsdc, swe, workloads
    params = swe.ModelParams(**workloads.EARTH)
    hier = mlsdc.build_hierarchy(params, 31, nf, 15, nc, grid_fine=(96, 48), grid_coarse=(48, 24))
    tag = f"ml{nf}{nc}_cs{ncs}"
    x = swe.PrognosticState(golden[f"{tag}_x"])
    sw_f, sw_c = mlsdc.initialize_mlsdc(x, hier)
    for _ in range(2):
        mlsdc.mlsdc_iteration(sw_f, sw_c, hier, dt, n_coarse_sweeps=ncs)
    y = sw_f.theta[-1].numpy()
    want = golden[f"{tag}_out"]
    for f in range(3):
        assert rel_err(y[f], want[f]) < 1e-9
    fc, cc = hier.fine.rhs.counters, hier.coarse.rhs.counters
    counts = [fc.solves, fc.implicit_evals, fc.explicit_evals, cc.solves, cc.implicit_evals,
              cc.explicit_evals]
    assert counts == list(golden[f"{tag}_counts"])


def test_config0_step_matches_reference():
    from paper_1805_07923_b200 import mlsdc, swe, workloads
    g = np.load(os.path.join(GOLDEN, "config0.npz"))
    params = swe.ModelParams(**workloads.EARTH)
    hier = mlsdc.build_hierarchy(params, 63, 3, 31, 2, grid_fine=(192, 96), grid_coarse=(96, 48))
    y = mlsdc.mlsdc_timestep(swe.PrognosticState(torch.as_tensor(g["x"]).cuda()), 600.0, 2, hier)
    y = y.numpy()
    for f in range(3):
        assert rel_err(y[f], g["out"][f]) < 1e-9
