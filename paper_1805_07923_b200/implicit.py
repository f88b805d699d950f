"""Drop-in for `swsdc.implicit` (reference implicit.py): per-mode implicit solve.

theta - beta F_I(theta) = b decouples per spectral mode into a scalar
vorticity division and a 2x2 (phi', delta) system (implicit.py:31-49); the
GPU kernel is csrc/spectral.cu:solve_kernel.  The determinant check and its
RuntimeError stay on the host, exactly as in the reference.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import _lib, spharm
from .spharm import _dev_guard, _ptr, _stream_ptr
from .swe import ModelParams, PrognosticState


@dataclasses.dataclass(frozen=True)
class ImplicitSolveContext:
    """beta = dt * qI_diag plus the mode eigenvalues (implicit.py:18-28)."""

    beta: float
    params: ModelParams
    lambdas: np.ndarray

    def __post_init__(self):
        if self.beta < 0:
            raise ValueError("implicit step must be non-negative")


def solve_implicit(b: PrognosticState, ctx: ImplicitSolveContext) -> PrognosticState:
    """Solve (I - beta F_I) theta = b mode by mode (implicit.py:31-49)."""
    beta = float(ctx.beta)
    lam = np.asarray(ctx.lambdas, dtype=float)
    nu, phi_bar = ctx.params.nu, ctx.params.phi_bar
    diag = 1.0 - beta * nu * lam
    det = diag * diag - beta * beta * lam * phi_bar
    if np.any(det <= 0.0):
        raise RuntimeError("implicit system is singular; invalid model parameters")
    R = b.truncation
    standard = spharm.laplacian_eigenvalues(R, ctx.params.radius)
    if lam.shape != standard.shape or not np.array_equal(lam, standard):
        raise ValueError("the GPU solve uses the Laplacian eigenvalues -s(s+1)/a^2 of the state")
    x = b.data.contiguous()
    out = torch.empty_like(x)
    nmat = int(np.prod(x.shape[:-3])) if x.dim() > 3 else 1
    cp = _lib.params_struct(ctx.params)
    with _dev_guard(x.device):
        _lib.check(_lib.load().swsdc_solve_implicit(R, ctypes.byref(cp), beta, _ptr(x), nmat,
                                                    _ptr(out), _stream_ptr(x.device)))
    return PrognosticState.from_tensor(out)
