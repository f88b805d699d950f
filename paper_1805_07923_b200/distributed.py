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

    def chunk_blocks(self, q: int, jh4: int, chunk: tuple[int, int] | None) -> tuple[int, int]:
        """4-pair blocks of rank q's chunk (c, C): its block range cut into C pieces
        (every rank uses the same C, so chunk c of one rank travels in the same
        collective as chunk c of every other rank; pieces may be empty)."""
        b0, b1 = self.block_bounds(q, jh4)
        if chunk is None:
            return b0, b1
        c, C = chunk
        n = b1 - b0
        return b0 + (n * c) // C, b0 + (n * (c + 1)) // C

    def chunk_lats(self, q: int, jh4: int, Jh: int, chunk: tuple[int, int] | None) -> tuple[int, int]:
        b0, b1 = self.chunk_blocks(q, jh4, chunk)
        return min(4 * b0, Jh), min(4 * b1, Jh)


class TorchExchanger:
    """Collectives over torch.distributed: NCCL all_to_all / all_gather /
    all_reduce between GPUs (over NVLink/NVSwitch); on gloo (the CPU tests,
    and several processes sharing one GPU in the GPU tests) paired
    isend/irecv, with device tensors staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.native = dist.get_backend(group) == "nccl"

    def all_to_all(self, sends: list[torch.Tensor], recv_shapes: list[tuple]) -> list[torch.Tensor]:
        dev = sends[0].device
        if self.native:
            recvs = [torch.empty(s, dtype=sends[0].dtype, device=dev) for s in recv_shapes]
            self.dist.all_to_all(recvs, [t.contiguous() for t in sends], group=self.group)
            return recvs
        host = [t.detach().to("cpu").contiguous() for t in sends]
        recvs = [torch.empty(s, dtype=sends[0].dtype) for s in recv_shapes]
        reqs = []
        for q in range(self.P):
            if q == self.rank:
                recvs[q].copy_(host[q])
            else:
                reqs.append(self.dist.isend(host[q], q, group=self.group))
                reqs.append(self.dist.irecv(recvs[q], q, group=self.group))
        for r in reqs:
            r.wait()
        return [t.to(dev) for t in recvs]

    def all_to_all_flat(self, sbuf: torch.Tensor, ssizes: list[int], rbuf: torch.Tensor,
                        rsizes: list[int]) -> torch.Tensor:
        """One all-to-all of contiguous per-peer segments (all_to_all_single with
        split sizes: one NCCL collective); gloo stages device buffers through host."""
        if self.native:
            self.dist.all_to_all_single(rbuf, sbuf, output_split_sizes=list(rsizes),
                                        input_split_sizes=list(ssizes), group=self.group)
            return rbuf
        hs = sbuf.detach().to("cpu")
        hr = torch.empty(rbuf.shape, dtype=rbuf.dtype)
        self.dist.all_to_all_single(hr, hs, output_split_sizes=list(rsizes),
                                    input_split_sizes=list(ssizes), group=self.group)
        rbuf.copy_(hr)
        return rbuf

    def all_gather(self, mine: torch.Tensor) -> list[torch.Tensor]:
        """Every rank's `mine` (equal shapes), in rank order."""
        if self.native:
            out = [torch.empty_like(mine) for _ in range(self.P)]
            self.dist.all_gather(out, mine.contiguous(), group=self.group)
            return out
        out = [torch.empty(mine.shape, dtype=mine.dtype) for _ in range(self.P)]
        self.dist.all_gather(out, mine.detach().to("cpu").contiguous(), group=self.group)
        return [t.to(mine.device) for t in out]

    def all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        """Elementwise max over ranks (in place on NCCL; returns the result)."""
        import torch.distributed as dist
        if self.native:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            return t
        h = t.detach().to("cpu")
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
        return h.to(t.device)


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

    def all_gather(self, mine):
        return self.all_to_all([mine] * self.P, [tuple(mine.shape)] * self.P)

    def all_to_all_flat(self, sbuf, ssizes, rbuf, rsizes):
        sends = list(torch.split(sbuf, list(ssizes)))
        got = self.all_to_all(sends, [(n,) for n in rsizes])
        torch.cat(got, out=rbuf)
        return rbuf

    def all_reduce_max(self, t):
        got = self.all_to_all([t] * self.P, [tuple(t.shape)] * self.P)
        return torch.stack(got).amax(dim=0)

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

def _blocks(arr: torch.Tensor, outer: int, rows: int, cols: int, inner: int, blocks,
            buf: torch.Tensor | None, scatter: bool) -> torch.Tensor:
    """swsdc_exchange_blocks: gather (scatter=False) blocks (row0, row_step, nrows,
    col0, col1) of arr[outer][rows][cols][inner] into one contiguous buffer, or
    scatter the buffer back -- one library launch."""
    nb = len(blocks)
    arrs = [(ctypes.c_int * nb)(*[b[i] for b in blocks]) for i in range(5)]
    n = sum(outer * b[2] * (b[4] - b[3]) * inner for b in blocks)
    if buf is None:
        buf = torch.empty(n, dtype=torch.float64, device=arr.device)
    if n == 0:
        return buf
    _lib.check(_lib.load().swsdc_exchange_blocks(_ptr(arr), outer, rows, cols, inner, nb, *arrs,
                                                 _ptr(buf), 1 if scatter else 0,
                                                 _stream_ptr(arr.device)))
    return buf


def _seg_sizes(outer, inner, blocks):
    return [outer * b[2] * (b[4] - b[3]) * inner for b in blocks]


def exchange_eo(ex, spec: ShardSpec, eo: torch.Tensor, R: int, Jh: int, jh4: int,
                chunk: tuple[int, int] | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """eo [m, 5, R+1, Jh, 4] with valid own rows -> same shape with ALL rows valid
    for this rank's latitude pairs.  Device tensors: one pack launch, one flat
    all-to-all, one unpack launch (swsdc_exchange_blocks); host tensors (the gloo
    CPU tests) take the equivalent torch slicing below.  chunk = (c, C) moves only
    piece c of every rank's latitude range (into `out`, shared by the C calls), so
    the grid stage of piece c can run while piece c + 1 is in flight."""
    P = spec.P
    if eo.is_cuda and hasattr(ex, "all_to_all_flat"):
        m, f = eo.shape[0], eo.shape[1]
        arr = eo.contiguous()
        nmine = len(range(spec.rank, R + 1, P))
        sblocks = [(spec.rank, P, nmine, *spec.chunk_lats(q, jh4, Jh, chunk)) for q in range(P)]
        j0, j1 = spec.chunk_lats(spec.rank, jh4, Jh, chunk)
        rblocks = [(p, P, len(range(p, R + 1, P)), j0, j1) for p in range(P)]
        sbuf = _blocks(arr, m * f, R + 1, Jh, 4, sblocks, None, False)
        rs = _seg_sizes(m * f, 4, rblocks)
        rbuf = torch.empty(sum(rs), dtype=torch.float64, device=eo.device)
        ex.all_to_all_flat(sbuf, _seg_sizes(m * f, 4, sblocks), rbuf, rs)
        if out is None:
            out = torch.empty_like(arr)
        _blocks(out, m * f, R + 1, Jh, 4, rblocks, rbuf, True)
        return out
    rows = spec.rows(R)
    sends, shapes = [], []
    m = eo.shape[0]
    for q in range(P):
        j0, j1 = spec.chunk_lats(q, jh4, Jh, chunk)
        sends.append(eo[:, :, rows, j0:j1, :])
    j0, j1 = spec.chunk_lats(spec.rank, jh4, Jh, chunk)
    for p in range(P):
        nrows = len(range(p, R + 1, P))
        shapes.append((m, eo.shape[1], nrows, j1 - j0, 4))
    recvs = ex.all_to_all(sends, shapes)
    if out is None:
        out = torch.empty_like(eo)
    for p in range(P):
        out[:, :, p:R + 1:P, j0:j1, :] = recvs[p]
    return out


def exchange_x(ex, spec: ShardSpec, x: torch.Tensor, R: int, jh4: int,
               chunk: tuple[int, int] | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """x [m, G, R+1, jh4, F] (fragment-native analysis input, F = 2*nc*4) valid for
    all rows on this rank's latitude blocks -> same shape valid for own rows on
    ALL latitude blocks (device tensors: library pack / flat all-to-all / unpack).
    chunk = (c, C): only piece c of every rank's block range (into `out`), sent
    while the grid stage works on piece c + 1."""
    P = spec.P
    if x.is_cuda and hasattr(ex, "all_to_all_flat"):
        m, G, F = x.shape[0], x.shape[1], x.shape[-1]
        arr = x.contiguous()
        b0, b1 = spec.chunk_blocks(spec.rank, jh4, chunk)
        sblocks = [(p, P, len(range(p, R + 1, P)), b0, b1) for p in range(P)]
        nmine = len(range(spec.rank, R + 1, P))
        rblocks = [(spec.rank, P, nmine, *spec.chunk_blocks(q, jh4, chunk)) for q in range(P)]
        sbuf = _blocks(arr, m * G, R + 1, jh4, F, sblocks, None, False)
        rs = _seg_sizes(m * G, F, rblocks)
        rbuf = torch.empty(sum(rs), dtype=torch.float64, device=x.device)
        ex.all_to_all_flat(sbuf, _seg_sizes(m * G, F, sblocks), rbuf, rs)
        if out is None:
            out = torch.empty_like(arr)
        _blocks(out, m * G, R + 1, jh4, F, rblocks, rbuf, True)
        return out
    sends, shapes = [], []
    b0, b1 = spec.chunk_blocks(spec.rank, jh4, chunk)
    for p in range(P):
        sends.append(x[:, :, p:R + 1:P, b0:b1, :])
    nrows = len(range(spec.rank, R + 1, P))
    for q in range(P):
        c0, c1 = spec.chunk_blocks(q, jh4, chunk)
        shapes.append(tuple(x.shape[:2]) + (nrows, c1 - c0, x.shape[-1]))
    recvs = ex.all_to_all(sends, shapes)
    if out is None:
        out = torch.empty_like(x)
    for q in range(P):
        c0, c1 = spec.chunk_blocks(q, jh4, chunk)
        out[:, :, spec.rank:R + 1:P, c0:c1, :] = recvs[q]
    return out


def gather_state(ex, spec: ShardSpec, data: torch.Tensor) -> torch.Tensor:
    """Assemble the full (…, 3, R+1, R+1) state from every rank's own rows: one
    all-gather of each rank's rows, padded to the largest rank's row count."""
    R = data.shape[-1] - 1
    nmax = len(range(0, R + 1, spec.P))
    mine = torch.zeros(tuple(data.shape[:-2]) + (nmax, R + 1), dtype=data.dtype,
                       device=data.device)
    own = data[..., spec.rows(R), :]
    mine[..., : own.shape[-2], :] = own
    got = ex.all_gather(mine)
    out = torch.empty_like(data)
    for q in range(spec.P):
        n = len(range(q, R + 1, spec.P))
        out[..., q:R + 1:spec.P, :] = got[q][..., :n, :]
    return out


def owned_nonfinite(spec: ShardSpec, data: torch.Tensor) -> torch.Tensor:
    """Device int32 flag: 1 if any owned row of `data` holds a non-finite value."""
    R = data.shape[-1] - 1
    own = torch.view_as_real(data[..., spec.rows(R), :])
    return (~torch.isfinite(own)).any().to(torch.int32)


# ----------------------------------------------------------------------------
# sharded right-hand side
# ----------------------------------------------------------------------------

class ShardedRHS(ShallowWaterRHS):
    """ShallowWaterRHS whose eval_f_e runs the staged, exchanged pipeline.

    Use it inside `row_filter(P, rank)` (ShardedMLSDC does this) so every other
    library call of the sweep (solve, F_I, combines, restriction, FAS,
    interpolation) is row-filtered too."""

    def __init__(self, plan, params, exchanger, spec: ShardSpec, include_nonlinear: bool = True,
                 chunks: int = 4):
        super().__init__(plan, params, include_nonlinear)
        self.ex, self.spec = exchanger, spec
        # pieces of each rank's latitude range: exchanges of one piece run on a side
        # stream while the grid stage works on another (1 = the unpipelined order)
        self.chunks = max(1, int(chunks))
        self._comm = None
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
        eo_v = eo.view(m, 5, R + 1, self.Jh, 4)
        xb = torch.empty(m * self.x_per, dtype=torch.float64, device=dev)
        groups = self.x_per // ((R + 1) * self.jh4 * 2 * self.nc * 4)
        xv = xb.view(m, groups, R + 1, self.jh4, 2 * self.nc * 4)
        C = self.chunks
        if C == 1 or not x.is_cuda:
            eo_full = exchange_eo(self.ex, self.spec, eo_v, R, self.Jh, self.jh4)
            j0, j1 = self.spec.lat_bounds(self.spec.rank, self.jh4, self.Jh)
            _lib.check(lib.swsdc_fe_grid(self.plan.handle, cp, nl, _ptr(eo_full), m, j0, j1,
                                         _ptr(xb), st))
            x_full = exchange_x(self.ex, self.spec, xv, R, self.jh4).contiguous()
        else:
            # Pipeline over C pieces of the latitude range: the side
            # stream carries pack -> all-to-all -> unpack of one piece while the main
            # stream runs the grid stage of another.  Every rank issues the same
            # sequence of collectives: E/O pieces 0..C-1, then the x piece behind each
            # grid piece.  Exposed communication: the first E/O piece and the last x
            # piece; the analysis (a reduction over all latitudes) waits for all of x.
            main = torch.cuda.current_stream(dev)
            if self._comm is None:
                self._comm = torch.cuda.Stream(device=dev)
            comm = self._comm
            eo_full = torch.empty_like(eo_v)
            x_full = torch.empty_like(xv)
            ready = torch.cuda.Event()
            ready.record(main)
            ev_eo = [torch.cuda.Event() for _ in range(C)]
            with torch.cuda.stream(comm):
                comm.wait_event(ready)
                for c in range(C):
                    exchange_eo(self.ex, self.spec, eo_v, R, self.Jh, self.jh4, (c, C), eo_full)
                    ev_eo[c].record(comm)
            for c in range(C):
                j0, j1 = self.spec.chunk_lats(self.spec.rank, self.jh4, self.Jh, (c, C))
                main.wait_event(ev_eo[c])
                if j1 > j0:
                    _lib.check(lib.swsdc_fe_grid(self.plan.handle, cp, nl, _ptr(eo_full), m, j0, j1,
                                                 _ptr(xb), st))
                done = torch.cuda.Event()
                done.record(main)
                with torch.cuda.stream(comm):
                    comm.wait_event(done)
                    exchange_x(self.ex, self.spec, xv, R, self.jh4, (c, C), x_full)
            fin = torch.cuda.Event()
            fin.record(comm)
            main.wait_event(fin)
        out = torch.empty_like(x)
        _lib.check(lib.swsdc_fe_analysis(self.plan.handle, cp, nl, _ptr(x_full), m, _ptr(out), st))
        return PrognosticState.from_tensor(out)


def sharded_hierarchy(params, r_fine, nodes_fine, r_coarse, nodes_coarse, exchanger,
                      spec: ShardSpec, grid_fine=None, grid_coarse=None, device=None,
                      include_nonlinear: bool = True, chunks: int = 4):
    """build_hierarchy with ShardedRHS on both levels."""
    from . import mlsdc
    base = mlsdc.build_hierarchy(params, r_fine, nodes_fine, r_coarse, nodes_coarse,
                                 include_nonlinear, grid_fine, grid_coarse, device)
    lv = []
    for level in (base.fine, base.coarse):
        rhs = ShardedRHS(level.plan, params, exchanger, spec, include_nonlinear, chunks)
        lv.append(mlsdc.Level(plan=level.plan, tables=level.tables, rhs=rhs))
    return mlsdc.TwoLevelHierarchy(fine=lv[0], coarse=lv[1], ops=base.ops)


def sharded_mlsdc_timestep(theta: PrognosticState, dt: float, n_iterations: int, hier,
                           spec: ShardSpec, n_coarse_sweeps: int = 1) -> PrognosticState:
    """mlsdc_timestep on this rank's rows (state rows of other ranks are stale)."""
    from . import mlsdc
    with row_filter(spec.P, spec.rank):
        return mlsdc.mlsdc_timestep(theta, dt, n_iterations, hier, n_coarse_sweeps)


def sharded_mlsdc_run(theta: PrognosticState, dt: float, n_iterations: int, hier,
                      spec: ShardSpec, n_steps: int, n_coarse_sweeps: int = 1,
                      flags: torch.Tensor | None = None) -> PrognosticState:
    """n_steps sharded steps with the reference's per-step finiteness contract
    (harness.py:257-258): after each step a device flag records whether any
    owned row went non-finite (no host sync inside the loop); the flags are
    max-reduced over ranks once at the end and the first bad step raises
    InstabilityError(step) on every rank."""
    from .stepper import InstabilityError
    dev = theta.data.device
    if flags is None:
        flags = torch.zeros(n_steps, dtype=torch.int32, device=dev)
    st = theta
    for k in range(n_steps):
        st = sharded_mlsdc_timestep(st, dt, n_iterations, hier, spec, n_coarse_sweeps)
        flags[k] = owned_nonfinite(spec, st.data)
    flags = hier.fine.rhs.ex.all_reduce_max(flags)
    bad = torch.nonzero(flags)
    if bad.numel():
        raise InstabilityError(int(bad[0]))
    return st
