"""m-sharded multi-GPU execution of the MLSDC-SH hot path.

One process (rank) per GPU.  Spectral data is sharded CYCLICALLY by zonal
wavenumber: rank p owns rows r with r % P == p.  That balances the
triangular Legendre work (rows carry R+2-r degrees) to O(P/R) and -- unlike
folding r with R-r -- keeps fine->coarse restriction / interpolation and
every other spectral-space operation local, because the coarse rows of a rank
are exactly its fine rows with r <= R_c.  The grid stage is sharded by
latitude pairs in blocks of 4 (one analysis B fragment).

Per F_E evaluation (swe.py:251-279):
    synthesis (own rows) -> all-to-all #1 (E/O of own rows for each rank's
    latitude pairs) -> grid stage (own pairs, all rows) -> all-to-all #2
    (weighted Fourier vectors of each rank's rows for own pairs) -> analysis +
    assembly (own rows).
The exchanges are NCCL all-to-alls over NVLink (torch.distributed); the
library's kernels honour a row filter so every spectral-space kernel touches
only owned rows.  Unowned rows of a rank's state arrays are never read and
hold stale data; `gather_state` assembles the full state.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .spharm import _ptr, _stream_ptr
from .swe import PrognosticState, ShallowWaterRHS


@contextlib.contextmanager
def row_filter(nranks: int, rank: int):
    """Make library kernels on this thread process only rows r % nranks == rank."""
    lib = _lib.load()
    _lib.check(lib.swsdc_set_row_filter(int(nranks), int(rank)))
    try:
        yield
    finally:
        _lib.check(lib.swsdc_set_row_filter(1, 0))


class ShardSpec:
    """Row and latitude ownership of one rank."""

    def __init__(self, nranks: int, rank: int):
        if not 0 <= rank < nranks:
            raise ValueError("rank out of range")
        self.P, self.rank = nranks, rank

    def rows(self, R: int) -> slice:
        return slice(self.rank, R + 1, self.P)

    def block_bounds(self, q: int, jh4: int) -> tuple[int, int]:
        """4-pair blocks [b0, b1) of rank q."""
        return (q * jh4) // self.P, ((q + 1) * jh4) // self.P

    def lat_bounds(self, q: int, jh4: int, Jh: int) -> tuple[int, int]:
        b0, b1 = self.block_bounds(q, jh4)
        return min(4 * b0, Jh), min(4 * b1, Jh)


class TorchExchanger:
    """all-to-all over torch.distributed: NCCL all_to_all between GPUs (one
    collective over NVLink/NVSwitch); on backends without all_to_all (gloo,
    the CPU tests) paired isend/irecv."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.native = dist.get_backend(group) == "nccl"

    def all_to_all(self, sends: list[torch.Tensor], recv_shapes: list[tuple]) -> list[torch.Tensor]:
        recvs = [torch.empty(s, dtype=sends[0].dtype, device=sends[0].device) for s in recv_shapes]
        sends = [t.contiguous() for t in sends]
        if self.native:
            self.dist.all_to_all(recvs, sends, group=self.group)
            return recvs
        reqs = []
        for q in range(self.P):
            if q == self.rank:
                recvs[q].copy_(sends[q])
            else:
                reqs.append(self.dist.isend(sends[q], q, group=self.group))
                reqs.append(self.dist.irecv(recvs[q], q, group=self.group))
        for r in reqs:
            r.wait()
        return recvs


class LocalExchanger:
    """P virtual ranks as threads of one process (one GPU): exchanges go
    through host-side barriers and device copies -- no kernel ever waits on
    another, so this is safe on a single GPU.  For tests and emulation."""

    def __init__(self, nranks: int):
        self.P = nranks
        self._barrier = threading.Barrier(nranks)
        self._slots = [None] * nranks

    def view(self, rank: int) -> "_LocalRank":
        return _LocalRank(self, rank)


class _LocalRank:
    def __init__(self, hub: LocalExchanger, rank: int):
        self.hub, self.P, self.rank = hub, hub.P, rank

    def all_to_all(self, sends, recv_shapes):
        hub = self.hub
        torch.cuda.synchronize() if sends and sends[0].is_cuda else None
        hub._slots[self.rank] = sends
        hub._barrier.wait()
        recvs = [hub._slots[q][self.rank].clone() for q in range(self.P)]
        for q, s in enumerate(recv_shapes):
            if tuple(recvs[q].shape) != tuple(s):
                raise RuntimeError(f"exchange shape mismatch from rank {q}: {recvs[q].shape} vs {s}")
        hub._barrier.wait()
        return recvs


# ----------------------------------------------------------------------------
# exchange packing (pure torch: unit-tested on CPU with gloo)
# ----------------------------------------------------------------------------

def exchange_eo(ex, spec: ShardSpec, eo: torch.Tensor, R: int, Jh: int, jh4: int) -> torch.Tensor:
    """eo [m, 5, R+1, Jh, 4] with valid own rows -> same shape with ALL rows valid
    for this rank's latitude pairs."""
    P = spec.P
    rows = spec.rows(R)
    sends, shapes = [], []
    m = eo.shape[0]
    for q in range(P):
        j0, j1 = spec.lat_bounds(q, jh4, Jh)
        sends.append(eo[:, :, rows, j0:j1, :])
    j0, j1 = spec.lat_bounds(spec.rank, jh4, Jh)
    for p in range(P):
        nrows = len(range(p, R + 1, P))
        shapes.append((m, eo.shape[1], nrows, j1 - j0, 4))
    recvs = ex.all_to_all(sends, shapes)
    out = torch.empty_like(eo)
    for p in range(P):
        out[:, :, p:R + 1:P, j0:j1, :] = recvs[p]
    return out


def exchange_x(ex, spec: ShardSpec, x: torch.Tensor, R: int, jh4: int) -> torch.Tensor:
    """x [m, G, R+1, jh4, F] (fragment-native analysis input, F = 2*nc*4) valid for
    all rows on this rank's latitude blocks -> same shape valid for own rows on
    ALL latitude blocks."""
    P = spec.P
    sends, shapes = [], []
    b0, b1 = spec.block_bounds(spec.rank, jh4)
    for p in range(P):
        sends.append(x[:, :, p:R + 1:P, b0:b1, :])
    nrows = len(range(spec.rank, R + 1, P))
    for q in range(P):
        c0, c1 = spec.block_bounds(q, jh4)
        shapes.append(tuple(x.shape[:2]) + (nrows, c1 - c0, x.shape[-1]))
    recvs = ex.all_to_all(sends, shapes)
    out = torch.empty_like(x)
    for q in range(P):
        c0, c1 = spec.block_bounds(q, jh4)
        out[:, :, spec.rank:R + 1:P, c0:c1, :] = recvs[q]
    return out


def gather_state(ex, spec: ShardSpec, data: torch.Tensor) -> torch.Tensor:
    """Assemble the full (…, 3, R+1, R+1) state from every rank's own rows."""
    R = data.shape[-1] - 1
    mine = data[..., spec.rows(R), :].contiguous()
    sends = [mine] * spec.P
    shapes = [tuple(data.shape[:-2]) + (len(range(q, R + 1, spec.P)), R + 1) for q in range(spec.P)]
    recvs = ex.all_to_all(sends, shapes)
    out = torch.empty_like(data)
    for q in range(spec.P):
        out[..., q:R + 1:spec.P, :] = recvs[q]
    return out


# ----------------------------------------------------------------------------
# sharded right-hand side
# ----------------------------------------------------------------------------

class ShardedRHS(ShallowWaterRHS):
    """ShallowWaterRHS whose eval_f_e runs the staged, exchanged pipeline.

    Use it inside `row_filter(P, rank)` (ShardedMLSDC does this) so every other
    library call of the sweep (solve, F_I, combines, restriction, FAS,
    interpolation) is row-filtered too."""

    def __init__(self, plan, params, exchanger, spec: ShardSpec, include_nonlinear: bool = True):
        super().__init__(plan, params, include_nonlinear)
        self.ex, self.spec = exchanger, spec
        lib = _lib.load()
        eo_n, x_n, nc, jh4 = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int()
        _lib.check(lib.swsdc_fe_layout(plan.handle, 1 if include_nonlinear else 0, 1,
                                       ctypes.byref(eo_n), ctypes.byref(x_n), ctypes.byref(nc),
                                       ctypes.byref(jh4)))
        self.eo_per = eo_n.value
        self.x_per = x_n.value
        self.nc, self.jh4 = nc.value, jh4.value
        self.Jh = (plan.grid.n_lat + 1) // 2

    def eval_f_e(self, state: PrognosticState) -> PrognosticState:
        self.counters.explicit_evals += 1
        self._check(state)
        lib = _lib.load()
        R = self.truncation
        x = state.data.contiguous()
        m = self._nmat(state)
        dev = x.device
        nl = 1 if self.include_nonlinear else 0
        cp = ctypes.byref(self._cparams)
        st = _stream_ptr(dev)
        eo = torch.empty(m * self.eo_per, dtype=torch.float64, device=dev)
        _lib.check(lib.swsdc_fe_synthesis(self.plan.handle, cp, _ptr(x), m, _ptr(eo), st))
        eo_full = exchange_eo(self.ex, self.spec, eo.view(m, 5, R + 1, self.Jh, 4), R, self.Jh,
                              self.jh4)
        j0, j1 = self.spec.lat_bounds(self.spec.rank, self.jh4, self.Jh)
        xb = torch.empty(m * self.x_per, dtype=torch.float64, device=dev)
        _lib.check(lib.swsdc_fe_grid(self.plan.handle, cp, nl, _ptr(eo_full), m, j0, j1, _ptr(xb),
                                     st))
        groups = self.x_per // ((R + 1) * self.jh4 * 2 * self.nc * 4)
        xv = xb.view(m, groups, R + 1, self.jh4, 2 * self.nc * 4)
        x_full = exchange_x(self.ex, self.spec, xv, R, self.jh4).contiguous()
        out = torch.empty_like(x)
        _lib.check(lib.swsdc_fe_analysis(self.plan.handle, cp, nl, _ptr(x_full), m, _ptr(out), st))
        return PrognosticState.from_tensor(out)


def sharded_hierarchy(params, r_fine, nodes_fine, r_coarse, nodes_coarse, exchanger,
                      spec: ShardSpec, grid_fine=None, grid_coarse=None, device=None,
                      include_nonlinear: bool = True):
    """build_hierarchy with ShardedRHS on both levels."""
    from . import mlsdc
    base = mlsdc.build_hierarchy(params, r_fine, nodes_fine, r_coarse, nodes_coarse,
                                 include_nonlinear, grid_fine, grid_coarse, device)
    lv = []
    for level in (base.fine, base.coarse):
        rhs = ShardedRHS(level.plan, params, exchanger, spec, include_nonlinear)
        lv.append(mlsdc.Level(plan=level.plan, tables=level.tables, rhs=rhs))
    return mlsdc.TwoLevelHierarchy(fine=lv[0], coarse=lv[1], ops=base.ops)


def sharded_mlsdc_timestep(theta: PrognosticState, dt: float, n_iterations: int, hier,
                           spec: ShardSpec, n_coarse_sweeps: int = 1) -> PrognosticState:
    """mlsdc_timestep on this rank's rows (state rows of other ranks are stale)."""
    from . import mlsdc
    with row_filter(spec.P, spec.rank):
        return mlsdc.mlsdc_timestep(theta, dt, n_iterations, hier, n_coarse_sweeps)
