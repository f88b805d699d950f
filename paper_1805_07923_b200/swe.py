"""Drop-in for `swsdc.swe` (reference swe.py) on a B200.

`PrognosticState` keeps (phi_prime, zeta, delta) as ONE device tensor of
shape (..., 3, R+1, R+1) complex128 (an optional leading member axis carries
ensembles); its algebra runs through the library's `combine` kernel.
`ShallowWaterRHS.eval_f_e` is the fused GPU pipeline
(synthesis -> grid products -> analysis -> assembly, csrc/) and
`eval_f_i` / `solve_implicit` are single elementwise kernels.  Counters are
incremented exactly where the reference increments them (swe.py:248, 257,
284).
"""

from __future__ import annotations

import ctypes
import math
import dataclasses

import numpy as np
import torch

from . import _lib, spharm
from .spharm import TransformPlan, _dev_guard, _ptr, _stream_ptr, _to_device


@dataclasses.dataclass(frozen=True)
class ModelParams:
    """Physical constants (swe.py:20-41); phi_bar = g * h_bar."""

    radius: float
    omega: float
    gravity: float
    nu: float
    h_bar: float

    def __post_init__(self):
        if self.radius <= 0 or self.gravity <= 0 or self.h_bar <= 0:
            raise ValueError("radius, gravity and h_bar must be positive")
        if self.nu < 0:
            raise ValueError("diffusion coefficient must be non-negative")

    @property
    def phi_bar(self) -> float:
        return self.gravity * self.h_bar


def combine(weights, tensors, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = sum_k w_k x_k on the device, skipping exactly-zero weights
    (sdc.py:211-220).  All tensors share shape and dtype complex128."""
    pairs = [(float(w), t) for w, t in zip(weights, tensors) if float(w) != 0.0]
    ref = tensors[0]
    if any(t.shape != ref.shape for t in tensors):
        raise ValueError("combine needs tensors of one shape")
    if out is None:
        out = torch.empty_like(ref)
    if not pairs:
        out.zero_()
        return out
    if len(pairs) > 32:
        raise ValueError("combine supports at most 32 weighted terms")
    lib = _lib.load()
    n = len(pairs)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for _, t in pairs])
    ws = (ctypes.c_double * n)(*[w for w, _ in pairs])
    with _dev_guard(ref.device):
        _lib.check(lib.swsdc_combine(n, ptrs, ws, ref.numel() * 2, _ptr(out),
                                     _stream_ptr(ref.device)))
    return out


def spec_combine(weights, tensors, r_out: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = sum_k w_k resize(x_k -> r_out), one launch; inputs may have
    different truncations (last two dims) but the same leading shape.
    Exactly-zero weights are skipped (sdc.py:211-220)."""
    pairs = [(float(w), t) for w, t in zip(weights, tensors) if float(w) != 0.0]
    ref = tensors[0]
    lead = tuple(ref.shape[:-2])
    if any(tuple(t.shape[:-2]) != lead for t in tensors):
        raise ValueError("spec_combine needs one leading shape")
    if out is None:
        out = torch.empty(lead + (r_out + 1, r_out + 1), dtype=torch.complex128, device=ref.device)
    if not pairs:
        out.zero_()
        return out
    if len(pairs) > 32:
        raise ValueError("spec_combine supports at most 32 weighted terms")
    n = len(pairs)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for _, t in pairs])
    ws = (ctypes.c_double * n)(*[w for w, _ in pairs])
    rin = (ctypes.c_int * n)(*[t.shape[-1] - 1 for _, t in pairs])
    nmat = math.prod(lead)
    with _dev_guard(ref.device):
        _lib.check(_lib.load().swsdc_spec_combine(n, ptrs, ws, rin, r_out, nmat, _ptr(out),
                                                  _stream_ptr(ref.device)))
    return out


def spec_combine_multi(jobs, r_out: int) -> list:
    """Several independent spec_combine sums [(weights, tensors, out or None), ...]
    in as few launches as the kernel's limits allow (16 outputs, 96 terms).
    Outputs may update one of their own inputs in place; no output may be
    another job's input.  Returns the output tensors in job order."""
    outs, batch = [], []
    prep = []
    for weights, tensors, out in jobs:
        pairs = [(float(w), t) for w, t in zip(weights, tensors) if float(w) != 0.0]
        ref = tensors[0]
        lead = tuple(ref.shape[:-2])
        if any(tuple(t.shape[:-2]) != lead for t in tensors):
            raise ValueError("spec_combine needs one leading shape")
        if out is None:
            out = torch.empty(lead + (r_out + 1, r_out + 1), dtype=torch.complex128,
                              device=ref.device)
        if len(pairs) > 32:
            raise ValueError("spec_combine supports at most 32 weighted terms")
        # in place with a unit self term and only coarser other terms: entries
        # beyond the other terms' truncation are unchanged, so skip them
        ext = r_out
        if pairs and pairs[0][1].data_ptr() == out.data_ptr() and pairs[0][0] == 1.0 \
                and pairs[0][1].shape[-1] - 1 == r_out and len(pairs) > 1:
            ext = max(t.shape[-1] - 1 for _, t in pairs[1:])
        prep.append((pairs, out, lead, ext))
        outs.append(out)
    if not prep:
        return outs
    lead0 = prep[0][2]
    if any(p[2] != lead0 for p in prep):
        raise ValueError("spec_combine_multi needs one leading shape across jobs")
    nmat = math.prod(lead0)
    dev = prep[0][1].device
    i = 0
    while i < len(prep):
        # greedy chunk within the kernel's limits
        group, terms = [], 0
        while i < len(prep) and len(group) < 16 and terms + len(prep[i][0]) <= 96:
            group.append(prep[i])
            terms += len(prep[i][0])
            i += 1
        nt = (ctypes.c_int * len(group))(*[len(p[0]) for p in group])
        flat = [pt for p in group for pt in p[0]]
        ptrs = (ctypes.c_void_p * max(1, len(flat)))(*[t.data_ptr() for _, t in flat])
        ws = (ctypes.c_double * max(1, len(flat)))(*[w for w, _ in flat])
        rin = (ctypes.c_int * max(1, len(flat)))(*[t.shape[-1] - 1 for _, t in flat])
        outp = (ctypes.c_void_p * len(group))(*[p[1].data_ptr() for p in group])
        exts = (ctypes.c_int * len(group))(*[p[3] for p in group])
        with _dev_guard(dev):
            _lib.check(_lib.load().swsdc_spec_combine_multi(len(group), nt, ptrs, ws, rin, r_out,
                                                            nmat, outp, exts, _stream_ptr(dev)))
    return outs


class PrognosticState:
    """Spectral state (phi_prime, zeta, delta) at one truncation (swe.py:44-125)."""

    __slots__ = ("data",)

    def __init__(self, phi_prime, zeta=None, delta=None):
        if zeta is None and delta is None:
            data, _ = _to_device(phi_prime, torch.complex128, _device_of(phi_prime))
            if data.dim() < 3 or data.shape[-3] != 3:
                raise ValueError("state tensor must have shape (..., 3, R+1, R+1)")
            self.data = data
            return
        dev = _device_of(phi_prime)
        parts = [_to_device(f, torch.complex128, dev)[0] for f in (phi_prime, zeta, delta)]
        if not (parts[0].shape == parts[1].shape == parts[2].shape):
            raise ValueError("prognostic fields must share one truncation")
        self.data = torch.stack(parts, dim=-3).contiguous()

    @classmethod
    def from_tensor(cls, data: torch.Tensor) -> "PrognosticState":
        st = cls.__new__(cls)
        st.data = data
        return st

    @classmethod
    def zeros(cls, truncation: int, device=None, members: int | None = None) -> "PrognosticState":
        dev = torch.device(device) if device is not None else spharm.default_device()
        shape = (3, truncation + 1, truncation + 1)
        if members is not None:
            shape = (members,) + shape
        return cls.from_tensor(torch.zeros(shape, dtype=torch.complex128, device=dev))

    @property
    def phi_prime(self) -> torch.Tensor:
        return self.data[..., 0, :, :]

    @property
    def zeta(self) -> torch.Tensor:
        return self.data[..., 1, :, :]

    @property
    def delta(self) -> torch.Tensor:
        return self.data[..., 2, :, :]

    @property
    def truncation(self) -> int:
        return self.data.shape[-1] - 1

    @property
    def device(self):
        return self.data.device

    def copy(self) -> "PrognosticState":
        return PrognosticState.from_tensor(self.data.clone())

    def __add__(self, other: "PrognosticState") -> "PrognosticState":
        _same(self, other)
        return PrognosticState.from_tensor(combine((1.0, 1.0), (self.data, other.data)))

    def __sub__(self, other: "PrognosticState") -> "PrognosticState":
        _same(self, other)
        return PrognosticState.from_tensor(combine((1.0, -1.0), (self.data, other.data)))

    def __mul__(self, scalar: float) -> "PrognosticState":
        return PrognosticState.from_tensor(combine((float(scalar),), (self.data,)))

    __rmul__ = __mul__

    def __iadd__(self, other: "PrognosticState") -> "PrognosticState":
        _same(self, other)
        combine((1.0, 1.0), (self.data, other.data), out=self.data)
        return self

    def fields(self):
        return self.phi_prime, self.zeta, self.delta

    def linf(self) -> float:
        return float(self.data.abs().max()) if self.data.numel() else 0.0

    def isfinite(self) -> bool:
        return bool(torch.isfinite(torch.view_as_real(self.data)).all())

    def truncated(self, truncation: int) -> "PrognosticState":
        return PrognosticState.from_tensor(spharm.truncate(self.data, truncation))

    def padded(self, truncation: int) -> "PrognosticState":
        return PrognosticState.from_tensor(spharm.pad(self.data, truncation))

    def numpy(self) -> np.ndarray:
        return self.data.cpu().numpy()


def _device_of(x):
    return x.device if isinstance(x, torch.Tensor) else spharm.default_device()


def _same(a: PrognosticState, b: PrognosticState) -> None:
    if a.data.shape != b.data.shape:
        raise ValueError("prognostic fields must share one truncation")


@dataclasses.dataclass
class DiagnosticVelocities:
    u: torch.Tensor
    v: torch.Tensor
    psi: torch.Tensor
    chi: torch.Tensor


@dataclasses.dataclass
class EvalCounters:
    """Running totals of solves and right-hand-side evaluations (swe.py:138-154)."""

    solves: int = 0
    implicit_evals: int = 0
    explicit_evals: int = 0

    def snapshot(self) -> "EvalCounters":
        return EvalCounters(self.solves, self.implicit_evals, self.explicit_evals)

    def since(self, other: "EvalCounters") -> "EvalCounters":
        return EvalCounters(self.solves - other.solves,
                            self.implicit_evals - other.implicit_evals,
                            self.explicit_evals - other.explicit_evals)


class ShallowWaterRHS:
    """Split right-hand sides at one truncation (swe.py:157-288)."""

    def __init__(self, plan: TransformPlan, params: ModelParams, include_nonlinear: bool = True):
        self.plan = plan
        self.params = params
        self.include_nonlinear = include_nonlinear
        self.counters = EvalCounters()
        self.truncation = plan.truncation
        self.lambdas = spharm.laplacian_eigenvalues(plan.truncation, params.radius)
        self._cparams = _lib.params_struct(params)
        dev = plan.device
        mu = torch.as_tensor(plan.grid.mu, device=dev)
        self._f_grid = (2.0 * params.omega * mu)[None, :]
        self._two_omega_over_a = 2.0 * params.omega / params.radius
        self._inv_cos2 = (1.0 / (1.0 - mu ** 2))[None, :]

    # -- diagnostics (swe.py:184-202) ------------------------------------------
    def cos_weighted_velocities(self, state: PrognosticState):
        a = self.params.radius
        psi = spharm.inv_laplacian(state.zeta, a)
        chi = spharm.inv_laplacian(state.delta, a)
        cu, cv = self.plan.synthesize_pair_cos_gradient(psi, chi)
        return cu * (1.0 / a), cv * (1.0 / a), psi, chi

    def helmholtz_velocities(self, state: PrognosticState) -> DiagnosticVelocities:
        cu, cv, psi, chi = self.cos_weighted_velocities(state)
        inv_cos = torch.as_tensor(1.0 / self.plan.grid.cos_lat, device=cu.device)[None, :]
        return DiagnosticVelocities(u=cu * inv_cos, v=cv * inv_cos, psi=psi, chi=chi)

    def div_curl(self, cos_u, cos_v):
        div, curl = self.plan.analyze_vector_div_curl(cos_u, cos_v)
        s = 1.0 / self.params.radius
        return div * s, curl * s

    # -- split right-hand sides -------------------------------------------------
    def _check(self, state: PrognosticState) -> None:
        if state.truncation != self.truncation:
            raise ValueError(
                f"state truncation {state.truncation} does not match RHS truncation {self.truncation}")

    def _nmat(self, state: PrognosticState) -> int:
        return int(np.prod(state.data.shape[:-3])) if state.data.dim() > 3 else 1

    def eval_l_g(self, state: PrognosticState) -> PrognosticState:
        """L_G: gravity-wave coupling + diffusion (swe.py:206-217), one kernel."""
        self._check(state)
        x = state.data.contiguous()
        out = torch.empty_like(x)
        with _dev_guard(x.device):
            _lib.check(_lib.load().swsdc_eval_fi(self.truncation, ctypes.byref(self._cparams),
                                                 _ptr(x), self._nmat(state), _ptr(out),
                                                 _stream_ptr(x.device)))
        return PrognosticState.from_tensor(out)

    def _fe(self, state: PrognosticState, nonlinear: bool) -> PrognosticState:
        self._check(state)
        x = state.data.contiguous()
        out = torch.empty_like(x)
        with _dev_guard(x.device):
            _lib.check(_lib.load().swsdc_eval_fe(self.plan.handle, ctypes.byref(self._cparams),
                                                 1 if nonlinear else 0, _ptr(x), self._nmat(state),
                                                 _ptr(out), _stream_ptr(x.device)))
        return PrognosticState.from_tensor(out)

    def eval_l_f(self, state: PrognosticState) -> PrognosticState:
        """Coriolis terms (swe.py:219-233) = the linear part of the fused F_E."""
        return self._fe(state, nonlinear=False)

    def eval_n(self, state: PrognosticState) -> PrognosticState:
        """Quadratic advection terms (swe.py:235-244), composed from transforms."""
        cu, cv, _, _ = self.cos_weighted_velocities(state)
        phi_grid = self.plan.synthesize(state.phi_prime)
        zeta_grid = self.plan.synthesize(state.zeta)
        div_phi, _ = self.div_curl(phi_grid * cu, phi_grid * cv)
        div_zeta, curl_zeta = self.div_curl(zeta_grid * cu, zeta_grid * cv)
        kinetic = 0.5 * (cu * cu + cv * cv) * self._inv_cos2
        lap_kinetic = spharm.laplacian(self.plan.analyze(kinetic), self.params.radius)
        return PrognosticState(-div_phi, -div_zeta, curl_zeta - lap_kinetic)

    def eval_f_i(self, state: PrognosticState) -> PrognosticState:
        """swe.py:246-249."""
        self.counters.implicit_evals += 1
        return self.eval_l_g(state)

    def eval_f_e(self, state: PrognosticState) -> PrognosticState:
        """Fused F_E = L_F + N (swe.py:251-279) on the GPU."""
        self.counters.explicit_evals += 1
        return self._fe(state, self.include_nonlinear)

    def solve_and_eval_fi(self, weights, tensors, beta: float):
        """Fused sweep node (sdc.py:196-205): b = sum_k w_k x_k, theta = solve(b, beta),
        f_i = F_I(theta) in ONE kernel.  Counts one solve and one implicit
        evaluation, like the reference's solve_implicit + eval_f_i."""
        if beta < 0:
            raise ValueError("implicit step must be non-negative")
        pairs = [(float(w), t) for w, t in zip(weights, tensors) if float(w) != 0.0]
        if len(pairs) > 32:
            raise ValueError("at most 32 terms")
        ref = tensors[0]
        theta = torch.empty_like(ref)
        fi = torch.empty_like(ref)
        n = len(pairs)
        ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for _, t in pairs])
        ws = (ctypes.c_double * n)(*[w for w, _ in pairs])
        nmat = int(np.prod(ref.shape[:-3])) if ref.dim() > 3 else 1
        with _dev_guard(ref.device):
            _lib.check(_lib.load().swsdc_sweep_node(self.truncation, ctypes.byref(self._cparams),
                                                    float(beta), n, ptrs, ws, nmat, _ptr(theta),
                                                    _ptr(fi), _stream_ptr(ref.device)))
        self.counters.solves += 1
        self.counters.implicit_evals += 1
        return PrognosticState.from_tensor(theta), PrognosticState.from_tensor(fi)

    def solve_implicit(self, b: PrognosticState, beta: float) -> PrognosticState:
        """swe.py:281-288."""
        from .implicit import ImplicitSolveContext, solve_implicit

        self.counters.solves += 1
        ctx = ImplicitSolveContext(beta=beta, params=self.params, lambdas=self.lambdas)
        return solve_implicit(b, ctx)
