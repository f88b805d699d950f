"""Drop-in for `swsdc.spharm` (reference spharm.py) on a B200.

Same names, argument meaning and exceptions as the reference module; the
transforms run on the GPU through libswsdc_b200.so (include/swsdc_b200.h).

Arrays: spectral coefficients are complex128 (..., R+1, R+1) dense [r, s]
with structural zeros for s < r; grids are float64 (..., n_lon, n_lat),
longitude-major, latitudes ascending in mu (spharm.py:3-17).  Methods accept
CUDA torch tensors (returned as CUDA tensors, zero host traffic) or numpy
arrays (copied to the device and back, for drop-in use).  Leading batch
dimensions are transformed in one launch sequence.

Host-side setup (Gauss nodes, grid metadata) is numpy, like the reference;
everything per transform is CUDA.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import dataclasses

import numpy as np
import torch

from . import _lib

__all__ = [
    "GaussianGrid",
    "TransformPlan",
    "build_gaussian_grid",
    "default_grid_shape",
    "gauss_legendre_nodes",
    "inv_laplacian",
    "laplacian",
    "laplacian_eigenvalues",
    "next_fast_size",
    "pad",
    "truncate",
    "zeros_coeffs",
]


def next_fast_size(n: int) -> int:
    """Smallest integer >= n with prime factors in {2, 3, 5} (spharm.py:40-49)."""
    m = n
    while True:
        k = m
        for p in (2, 3, 5):
            while k % p == 0:
                k //= p
        if k == 1:
            return m
        m += 1


def gauss_legendre_nodes(n: int, tol: float = 1e-14, max_iter: int = 100):
    """Gauss-Legendre nodes and weights on [-1, 1] (spharm.py:52-86).

    Host setup.  Newton on the Legendre recurrence from the guesses
    cos(pi (k - 1/4)/(n + 1/2)), same operation order as the reference, so the
    nodes are bitwise identical to it (tests/test_grid.py).
    """
    if n < 1:
        raise ValueError(f"need at least one node, got {n}")
    x = np.cos(np.pi * (np.arange(1, n + 1) - 0.25) / (n + 0.5))
    done = np.zeros(n, dtype=bool)
    dp = np.empty_like(x)
    for _ in range(max_iter):
        p0 = np.ones_like(x)
        p1 = x.copy()
        for deg in range(2, n + 1):
            p0, p1 = p1, ((2 * deg - 1) * x * p1 - (deg - 1) * p0) / deg
        dp = n * (x * p1 - p0) / (x * x - 1.0)
        dx = p1 / dp
        x -= dx
        done = np.abs(dx) <= tol
        if done.all():
            break
    if not done.all():
        raise RuntimeError(f"Gauss-Legendre root search failed to converge for n={n}")
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    order = np.argsort(x)
    x, w = x[order], w[order]
    x = 0.5 * (x - x[::-1])
    w = 0.5 * (w + w[::-1])
    return x, w


@dataclasses.dataclass(frozen=True)
class GaussianGrid:
    """Equispaced longitudes and Gaussian latitudes (spharm.py:89-118)."""

    n_lon: int
    n_lat: int
    mu: np.ndarray
    w: np.ndarray

    @property
    def lon(self) -> np.ndarray:
        return 2.0 * np.pi * np.arange(self.n_lon) / self.n_lon

    @property
    def lat(self) -> np.ndarray:
        return np.arcsin(self.mu)

    @property
    def cos_lat(self) -> np.ndarray:
        return np.sqrt(1.0 - self.mu * self.mu)

    def quad_mean(self, field) -> float:
        """Area-weighted global mean of a (n_lon, n_lat) field."""
        if isinstance(field, torch.Tensor):
            w = torch.as_tensor(self.w, device=field.device)
            return float((field * w).sum() / (2.0 * self.n_lon))
        return float(np.sum(field * self.w) / (2.0 * self.n_lon))


def build_gaussian_grid(n_lat: int, n_lon: int | None = None) -> GaussianGrid:
    """spharm.py:121-127."""
    mu, w = gauss_legendre_nodes(n_lat)
    if n_lon is None:
        n_lon = next_fast_size(2 * n_lat)
    return GaussianGrid(n_lon=n_lon, n_lat=n_lat, mu=mu, w=w)


def default_grid_shape(truncation: int) -> tuple[int, int]:
    """Dealiased (n_lon, n_lat) for truncation R (spharm.py:130-138)."""
    return next_fast_size(3 * truncation + 1), -(-(3 * truncation + 1) // 2)


# ----------------------------------------------------------------------------
# device-array helpers
# ----------------------------------------------------------------------------

def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1805_07923_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_device(x, dtype, device):
    """(tensor on device, contiguous, dtype) and whether the input was host numpy."""
    if isinstance(x, torch.Tensor):
        if x.device != device:
            x = x.to(device)
        if x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x), dtype=np.complex128 if dtype == torch.complex128 else np.float64)
    return torch.from_numpy(arr).to(device), True


def _is_pinned_host(x) -> bool:
    return isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.is_pinned()


def upload_coeffs(host: torch.Tensor, out: torch.Tensor | None = None, device=None) -> torch.Tensor:
    """Page-locked host coefficients (..., R+1, R+1) complex128 -> device tensor.

    Only the s >= r triangle that the reference layout populates crosses PCIe
    (a zero-copy kernel, half the bytes of a dense copy); the device copy's lower
    triangle is zero.  Asynchronous on the current stream, like
    `Tensor.to(non_blocking=True)`."""
    if not _is_pinned_host(host):
        raise ValueError("upload_coeffs needs a page-locked (pinned) host tensor")
    if host.dtype != torch.complex128 or not host.is_contiguous():
        raise ValueError("upload_coeffs needs a contiguous complex128 tensor")
    if host.dim() < 2 or host.shape[-1] != host.shape[-2]:
        raise ValueError(f"coefficient array of shape {tuple(host.shape)} is not (..., R+1, R+1)")
    device = torch.device(device) if device is not None else (
        out.device if out is not None else torch.device("cuda", torch.cuda.current_device()))
    if out is None:
        out = torch.empty(host.shape, dtype=torch.complex128, device=device)
    elif out.shape != host.shape or out.dtype != torch.complex128 or not out.is_contiguous():
        raise ValueError("out has the wrong shape or layout")
    R = host.shape[-1] - 1
    nmat = host.numel() // ((R + 1) * (R + 1))
    with _dev_guard(out.device):
        _lib.check(_lib.load().swsdc_upload_coeffs(_ptr(host), R, nmat, _ptr(out),
                                                   _stream_ptr(out.device)))
    return out


def download_coeffs(dev: torch.Tensor, out: torch.Tensor, write_lower: bool = True) -> torch.Tensor:
    """Device coefficients (..., R+1, R+1) -> page-locked host tensor `out` by the
    copy engine, asynchronous on the current stream.  write_lower=False sends
    (about) only the s >= r triangle, half the PCIe bytes: entries of `out` below
    it are either left untouched or receive the device's values -- for results
    streamed into a reused, zero-initialised buffer, where they stay zero."""
    if not _is_pinned_host(out):
        raise ValueError("download_coeffs needs a page-locked (pinned) host `out`")
    if (dev.dtype != torch.complex128 or out.dtype != torch.complex128 or not dev.is_cuda
            or not dev.is_contiguous() or not out.is_contiguous() or dev.shape != out.shape):
        raise ValueError("download_coeffs needs contiguous complex128 tensors of one shape")
    if dev.dim() < 2 or dev.shape[-1] != dev.shape[-2]:
        raise ValueError(f"coefficient array of shape {tuple(dev.shape)} is not (..., R+1, R+1)")
    R = dev.shape[-1] - 1
    nmat = dev.numel() // ((R + 1) * (R + 1))
    with _dev_guard(dev.device):
        _lib.check(_lib.load().swsdc_download_coeffs(_ptr(dev), R, nmat, _ptr(out),
                                                     1 if write_lower else 0,
                                                     _stream_ptr(dev.device)))
    return out


def _out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(device) -> int:
    """Raw cudaStream_t of the current stream on `device` (an int: ctypes converts
    it for c_void_p arguments); the cheap path avoids building a Stream object,
    which dominated the host cost of small calls."""
    idx = device.index
    if idx is None:
        idx = torch.cuda.current_device()
    if _raw_stream is not None:
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _dev_guard(device):
    """Make `device` current for the library's launches; a no-op (no context
    switch) when it already is."""
    if device.index is None or device.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(device)


class TransformPlan:
    """GPU transform plan at a fixed triangular truncation (spharm.py:182-300).

    Holds no dense (R+1, R+1, J) tables: the device plan keeps recurrence
    coefficients and per-chunk checkpoint seeds (csrc/legendre.cu).  Immutable
    after construction; one plan serialises its own scratch workspace, so use
    one plan per concurrent CUDA stream.
    """

    def __init__(self, grid: GaussianGrid, truncation: int, device=None):
        if truncation < 0:
            raise ValueError("truncation must be non-negative")
        if grid.n_lon < 2 * truncation + 1:
            raise ValueError(
                f"n_lon={grid.n_lon} cannot carry zonal wavenumbers up to {truncation}"
            )
        self.grid = grid
        self.truncation = truncation
        self.device = torch.device(device) if device is not None else default_device()
        lib = _lib.load()
        mu = np.ascontiguousarray(grid.mu, dtype=np.float64)
        w = np.ascontiguousarray(grid.w, dtype=np.float64)
        handle = ctypes.c_void_p()
        with _dev_guard(self.device):
            _lib.check(lib.swsdc_plan_create(
                truncation, grid.n_lon, grid.n_lat, mu.ctypes.data_as(ctypes.c_void_p),
                w.ctypes.data_as(ctypes.c_void_p), ctypes.byref(handle)))
        self._handle = handle
        self._lib = lib
        self._r = np.arange(truncation + 1)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.swsdc_plan_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    def reserve(self, fields: int) -> None:
        """Pre-size the scratch workspace (needed before CUDA graph capture)."""
        with _dev_guard(self.device):
            _lib.check(self._lib.swsdc_plan_reserve(self._handle, int(fields)))

    # -- shape helpers ------------------------------------------------------
    def _grid_in(self, field):
        t, host = _to_device(field, torch.float64, self.device)
        if tuple(t.shape[-2:]) != (self.grid.n_lon, self.grid.n_lat) or t.dim() < 2:
            raise ValueError(
                f"field shape {tuple(t.shape)} does not match grid "
                f"({self.grid.n_lon}, {self.grid.n_lat})"
            )
        return t, host

    def _coeff_in(self, coeffs):
        if (_is_pinned_host(coeffs) and coeffs.dtype == torch.complex128 and coeffs.is_contiguous()
                and coeffs.dim() >= 2 and coeffs.shape[-1] == coeffs.shape[-2]):
            t, host = upload_coeffs(coeffs, device=self.device), False
        else:
            t, host = _to_device(coeffs, torch.complex128, self.device)
        if t.dim() < 2 or t.shape[-1] != t.shape[-2]:
            raise ValueError(f"coefficient array of shape {tuple(t.shape)} is not (..., R+1, R+1)")
        r_in = t.shape[-1] - 1
        if r_in > self.truncation:
            raise ValueError(
                f"coefficients at truncation {r_in} exceed plan truncation {self.truncation}"
            )
        return t, host, r_in

    # -- public transforms (spharm.py:254-300) ------------------------------
    def analyze(self, field, out: torch.Tensor | None = None):
        """Grid field (..., n_lon, n_lat) -> coefficients (..., R+1, R+1).
        `out` (optional, contiguous complex128) receives the result in place: a CUDA
        tensor, or a page-locked host tensor filled by an asynchronous copy on the
        current stream (synchronize before reading it)."""
        g, host = self._grid_in(field)
        lead = g.shape[:-2]
        nb = math.prod(lead)
        R = self.truncation
        target = out
        if out is not None and (tuple(out.shape) != tuple(lead) + (R + 1, R + 1)
                                or not out.is_contiguous() or out.dtype != torch.complex128):
            raise ValueError("out has the wrong shape or layout")
        if out is not None and out.device.type == "cpu":
            if not out.is_pinned():
                raise ValueError("a host `out` must be page-locked (pinned)")
            out = None
        if out is None:
            out = torch.empty(lead + (R + 1, R + 1), dtype=torch.complex128, device=self.device)
        with _dev_guard(self.device):
            _lib.check(self._lib.swsdc_analyze(self._handle, _ptr(g), nb, _ptr(out),
                                               _stream_ptr(self.device)))
            if target is not None and target.device.type == "cpu":
                target.copy_(out, non_blocking=True)
                return target
        return _out(out, host)

    def synthesize(self, coeffs, out: torch.Tensor | None = None):
        """Coefficients (..., R_in+1, R_in+1), R_in <= R -> real grid (..., n_lon, n_lat).
        `out` (optional, CUDA, contiguous) receives the result in place."""
        c, host, r_in = self._coeff_in(coeffs)
        lead = c.shape[:-2]
        nb = math.prod(lead)
        shape = tuple(lead) + (self.grid.n_lon, self.grid.n_lat)
        if out is None:
            out = torch.empty(shape, dtype=torch.float64, device=self.device)
        elif tuple(out.shape) != shape or not out.is_contiguous():
            raise ValueError("out has the wrong shape or layout")
        with _dev_guard(self.device):
            _lib.check(self._lib.swsdc_synthesize(self._handle, _ptr(c), r_in, nb, _ptr(out),
                                                  _stream_ptr(self.device)))
        return _out(out, host)

    def synthesize_pair_cos_gradient(self, psi, chi):
        """U = u cos(phi), V = v cos(phi) on the unit sphere from psi, chi."""
        p, host, r_in = self._coeff_in(psi)
        c, _, r_in2 = self._coeff_in(chi)
        if p.shape != c.shape:
            raise ValueError("psi and chi must share one shape")
        lead = p.shape[:-2]
        nb = math.prod(lead)
        shape = lead + (self.grid.n_lon, self.grid.n_lat)
        u = torch.empty(shape, dtype=torch.float64, device=self.device)
        v = torch.empty(shape, dtype=torch.float64, device=self.device)
        with _dev_guard(self.device):
            _lib.check(self._lib.swsdc_synthesize_uv(self._handle, _ptr(p), _ptr(c), r_in, nb,
                                                     _ptr(u), _ptr(v), _stream_ptr(self.device)))
        return _out(u, host), _out(v, host)

    def analyze_vector_div_curl(self, cos_u, cos_v):
        """Spectral (div, curl) on the unit sphere from cos-weighted components."""
        u, host = self._grid_in(cos_u)
        v, _ = self._grid_in(cos_v)
        if u.shape != v.shape:
            raise ValueError("cos_u and cos_v must share one shape")
        lead = u.shape[:-2]
        nb = math.prod(lead)
        R = self.truncation
        div = torch.empty(lead + (R + 1, R + 1), dtype=torch.complex128, device=self.device)
        curl = torch.empty_like(div)
        with _dev_guard(self.device):
            _lib.check(self._lib.swsdc_analyze_divcurl(self._handle, _ptr(u), _ptr(v), nb,
                                                       _ptr(div), _ptr(curl),
                                                       _stream_ptr(self.device)))
        return _out(div, host), _out(curl, host)


# ----------------------------------------------------------------------------
# spectral operators (spharm.py:303-349)
# ----------------------------------------------------------------------------

def zeros_coeffs(truncation: int, device=None) -> torch.Tensor:
    dev = torch.device(device) if device is not None else default_device()
    return torch.zeros((truncation + 1, truncation + 1), dtype=torch.complex128, device=dev)


def laplacian_eigenvalues(truncation: int, radius: float) -> np.ndarray:
    """-s(s+1)/a^2, shape (R+1,) (host table, spharm.py:307-310)."""
    s = np.arange(truncation + 1, dtype=float)
    return -s * (s + 1.0) / (radius * radius)


def _laplacian(coeffs, radius: float, inverse: int):
    if radius <= 0:
        raise ValueError("radius must be positive")
    c, host = _to_device(coeffs, torch.complex128, _dev_of(coeffs))
    c = c.contiguous()
    out = torch.empty_like(c)
    lib = _lib.load()
    with _dev_guard(c.device):
        _lib.check(lib.swsdc_laplacian(_ptr(c), _ptr(out), c.shape[-1] - 1,
                                       math.prod(c.shape[:-2]), float(radius), inverse,
                                       _stream_ptr(c.device)))
    return _out(out, host)


def laplacian(coeffs, radius: float):
    """Multiply by -s(s+1)/a^2 (spharm.py:313-317); one library kernel."""
    return _laplacian(coeffs, radius, 0)


def inv_laplacian(coeffs, radius: float):
    """Inverse Laplacian with the s = 0 column gauged to zero (spharm.py:320-328),
    rounded as numpy's complex-by-real division; one library kernel."""
    return _laplacian(coeffs, radius, 1)


def _dev_of(x):
    return x.device if isinstance(x, torch.Tensor) else default_device()


def _resize(coeffs, r_out: int):
    c, host = _to_device(coeffs, torch.complex128, _dev_of(coeffs))
    r_in = c.shape[-1] - 1
    lead = c.shape[:-2]
    nmat = math.prod(lead)
    out = torch.empty(lead + (r_out + 1, r_out + 1), dtype=torch.complex128, device=c.device)
    lib = _lib.load()
    with _dev_guard(c.device):
        _lib.check(lib.swsdc_resize(_ptr(c), r_in, _ptr(out), r_out, nmat, _stream_ptr(c.device)))
    return _out(out, host)


def truncate(coeffs, truncation: int):
    """Keep r, s <= R_c (spharm.py:331-336)."""
    r_in = coeffs.shape[-1] - 1
    if truncation > r_in:
        raise ValueError(f"cannot truncate R={r_in} to larger R={truncation}")
    return _resize(coeffs, truncation)


def pad(coeffs, truncation: int):
    """Zero-embed into a larger truncation (spharm.py:339-349)."""
    r_in = coeffs.shape[-1] - 1
    if truncation < r_in:
        raise ValueError(f"cannot pad R={r_in} to smaller R={truncation}")
    return _resize(coeffs, truncation)
