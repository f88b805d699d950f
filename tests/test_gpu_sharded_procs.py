"""m-sharded MLSDC through TorchExchanger with REAL processes: 2 ranks share
cuda:0 over a gloo group (exchanges staged through host memory, so no kernel
of one rank waits on the other's).  A full MLSDC(5,3) step with two coarse
sweeps, gathered with all_gather, must match the unsharded oracle; a blown-up
state must raise InstabilityError(step) on every rank via the per-step
finiteness flag and its all-reduce (harness.py:257-258)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_07923_b200 import distributed as D
        from paper_1805_07923_b200 import stepper, swe, workloads
        torch.cuda.set_device(0)
        params = swe.ModelParams(**workloads.EARTH)
        ex = D.TorchExchanger()
        spec = D.ShardSpec(world, rank)
        hier = D.sharded_hierarchy(params, 31, 5, 15, 3, ex, spec, grid_fine=(96, 48),
                                   grid_coarse=(48, 24))
        x = workloads.seeded_state(31, 2)
        st = swe.PrognosticState(torch.as_tensor(x).cuda())
        y = D.sharded_mlsdc_run(st, 240.0, 2, hier, spec, 2, n_coarse_sweeps=2)
        full = D.gather_state(ex, spec, y.data).cpu().numpy()
        blown = None
        try:
            D.sharded_mlsdc_run(swe.PrognosticState(torch.as_tensor(x * 1e30).cuda()), 3600.0, 2,
                                hier, spec, 30)
        except stepper.InstabilityError as e:
            blown = e.step
        q.put((rank, full, blown, None))
    except Exception as e:  # surfaced by the parent
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_process_sharded_step_matches_oracle():
    import swsdc_oracle as orc
    from conftest import rel_err
    from paper_1805_07923_b200 import workloads
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, full, blown, err = q.get(timeout=600)
        res[rank] = (full, blown, err)
    for p in procs:
        p.join(60)
    for rank in range(2):
        assert res[rank][2] is None, res[rank][2]
    oh = orc.OracleHierarchy(orc.OracleLevel(31, 5, orc.OracleParams(**workloads.EARTH), (96, 48)),
                             orc.OracleLevel(15, 3, orc.OracleParams(**workloads.EARTH), (48, 24)))
    want = workloads.seeded_state(31, 2)
    for _ in range(2):
        want = orc.mlsdc_step(want, 240.0, 2, oh, coarse_sweeps=2)
    for rank in range(2):
        full, blown, _ = res[rank]
        for f in range(3):
            assert rel_err(full[f], want[f]) < 1e-9
        assert blown is not None and 0 <= blown < 30
    assert res[0][1] == res[1][1]   # every rank reports the same first bad step
