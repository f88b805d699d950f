"""m-sharding host logic with a real 2-rank torch.distributed (gloo) group on
the CPU: row/latitude ownership, both all-to-all exchange layouts of the
sharded F_E pipeline, and state gathering (paper_1805_07923_b200/distributed.py)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_1805_07923_b200.distributed import (ShardSpec, TorchExchanger, exchange_eo, exchange_x,
                                               gather_state)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _eo_value(m, f, r, jh, c):
    return 1e6 * m + 1e4 * f + 10.0 * r + jh + 0.1 * c


def _worker(rank, world, port, R, Jh, fails):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = ShardSpec(world, rank)
        ex = TorchExchanger()
        jh4 = (Jh + 3) // 4
        m = 2
        # --- exchange #1: each rank holds E/O only for its rows (others poisoned)
        idx = torch.meshgrid(torch.arange(m), torch.arange(5), torch.arange(R + 1), torch.arange(Jh),
                             torch.arange(4), indexing="ij")
        truth = _eo_value(*[t.double() for t in idx])
        eo = torch.full_like(truth, float("nan"))
        eo[:, :, rank:R + 1:world] = truth[:, :, rank:R + 1:world]
        full = exchange_eo(ex, spec, eo, R, Jh, jh4)
        j0, j1 = spec.lat_bounds(rank, jh4, Jh)
        assert torch.equal(full[:, :, :, j0:j1], truth[:, :, :, j0:j1]), "eo exchange"
        # --- exchange #2: x valid for all rows on own latitude blocks only
        F = 2 * 8 * 4
        xt = torch.arange(m * 1 * (R + 1) * jh4 * F, dtype=torch.float64).view(m, 1, R + 1, jh4, F)
        x = torch.full_like(xt, float("nan"))
        b0, b1 = spec.block_bounds(rank, jh4)
        x[:, :, :, b0:b1] = xt[:, :, :, b0:b1]
        xf = exchange_x(ex, spec, x, R, jh4)
        assert torch.equal(xf[:, :, rank:R + 1:world], xt[:, :, rank:R + 1:world]), "x exchange"
        # --- pipelined form: C pieces of every rank's latitude range, one collective each,
        #     assembled into one buffer (C = 5 leaves some pieces empty at small Jh)
        for C in (2, 3, 5):
            full_c = torch.full_like(truth, float("nan"))
            xf_c = torch.full_like(xt, float("nan"))
            for c in range(C):
                exchange_eo(ex, spec, eo, R, Jh, jh4, (c, C), full_c)
                exchange_x(ex, spec, x, R, jh4, (c, C), xf_c)
            assert torch.equal(full_c[:, :, :, j0:j1], truth[:, :, :, j0:j1]), f"eo pieces C={C}"
            assert torch.equal(xf_c[:, :, rank:R + 1:world], xt[:, :, rank:R + 1:world]), f"x pieces C={C}"
            pieces = [spec.chunk_blocks(rank, jh4, (c, C)) for c in range(C)]
            assert pieces[0][0] == b0 and pieces[-1][1] == b1
            assert all(pieces[c][1] == pieces[c + 1][0] for c in range(C - 1))
        # --- gather_state
        st = torch.randn(3, 3, R + 1, R + 1, dtype=torch.complex128, generator=torch.Generator().manual_seed(7))
        mine = torch.full_like(st, complex(float("nan"), 0.0))
        mine[..., rank:R + 1:world, :] = st[..., rank:R + 1:world, :]
        got = gather_state(ex, spec, mine)
        assert torch.equal(got, st), "gather_state"
        # --- flat all-to-all (the device path's single collective with split sizes)
        ssizes = [q + 1 + rank for q in range(world)]        # to q: q+1+rank values
        rsizes = [rank + 1 + p for p in range(world)]        # from p: rank+1+p values
        sbuf = torch.cat([torch.full((n,), 100.0 * rank + q, dtype=torch.float64)
                          for q, n in enumerate(ssizes)])
        rbuf = torch.empty(sum(rsizes), dtype=torch.float64)
        ex.all_to_all_flat(sbuf, ssizes, rbuf, rsizes)
        want = torch.cat([torch.full((n,), 100.0 * p + rank, dtype=torch.float64)
                          for p, n in enumerate(rsizes)])
        assert torch.equal(rbuf, want), "flat all-to-all"
        # --- per-step finiteness flag: a NaN in one rank's own rows reaches every rank
        from paper_1805_07923_b200.distributed import owned_nonfinite
        clean = owned_nonfinite(spec, st)
        assert int(ex.all_reduce_max(clean.view(1))[0]) == 0, "finite flag"
        dirty = st.clone()
        dirty[0, 0, 1, 2] = complex(float("nan"), 0.0)   # row 1 belongs to rank 1 % world
        flag = owned_nonfinite(spec, dirty)
        assert int(flag) == (1 if rank == 1 % world else 0), "own-row flag"
        assert int(ex.all_reduce_max(flag.view(1))[0]) == 1, "flag all-reduce"
        # --- ownership covers every row / latitude exactly once
        rows = sorted(r for q in range(world) for r in range(R + 1)[ShardSpec(world, q).rows(R)])
        assert rows == list(range(R + 1))
        lats = sorted(j for q in range(world) for j in range(*spec.lat_bounds(q, jh4, Jh)))
        assert lats == list(range(Jh))
    except AssertionError as e:
        fails.put(f"rank {rank}: {e}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("R,Jh", [(31, 24), (15, 12), (10, 9)])
def test_sharded_exchanges_gloo_world2(R, Jh):
    ctx = mp.get_context("spawn")
    fails = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, R, Jh, fails)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not fails.empty():
        errs.append(fails.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
