"""m-sharded MLSDC (distributed.py) on ONE GPU: P virtual ranks run as threads
with host-side exchanges (no kernel waits on another); the gathered state must
match the unsharded oracle step.  chunks > 1: the F_E exchanges travel in pieces
of the latitude range on a side stream while the grid stage works on other pieces
(chunks = 7 leaves some pieces empty on the coarse level's 6 blocks)."""

import threading

import numpy as np
import pytest
import torch

import swsdc_oracle as orc
from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P,chunks", [(2, 4), (3, 2), (2, 1), (3, 7)])
def test_sharded_mlsdc_step_matches_oracle(P, chunks):
    from paper_1805_07923_b200 import distributed as D
    from paper_1805_07923_b200 import swe, workloads
    params = swe.ModelParams(**workloads.EARTH)
    x = workloads.seeded_state(31, 2)
    hub = D.LocalExchanger(P)
    results, errors = [None] * P, []

    def run(rank):
        try:
            ex = hub.view(rank)
            spec = D.ShardSpec(P, rank)
            hier = D.sharded_hierarchy(params, 31, 5, 15, 3, ex, spec, grid_fine=(96, 48),
                                       grid_coarse=(48, 24), chunks=chunks)
            st = swe.PrognosticState(torch.as_tensor(x).cuda())
            y = D.sharded_mlsdc_timestep(st, 240.0, 2, hier, spec, n_coarse_sweeps=2)
            results[rank] = D.gather_state(ex, spec, y.data).cpu().numpy()
        except Exception as e:  # surface thread failures
            errors.append(repr(e))
            hub._barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errors, errors
    oh = orc.OracleHierarchy(orc.OracleLevel(31, 5, orc.OracleParams(**workloads.EARTH), (96, 48)),
                             orc.OracleLevel(15, 3, orc.OracleParams(**workloads.EARTH), (48, 24)))
    want = orc.mlsdc_step(x, 240.0, 2, oh, coarse_sweeps=2)
    for rank in range(P):
        for f in range(3):
            assert rel_err(results[rank][f], want[f]) < 1e-9
