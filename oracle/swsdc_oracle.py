"""CPU oracle for the MLSDC-SH hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 path.  It is a numpy
restatement of the reference algorithm in `/root/reference/pkg/src/swsdc/`
(spharm.py, swe.py, implicit.py, sdc.py, mlsdc.py); every function names the
reference lines it follows.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product package (`paper_1805_07923_b200`) never imports it: the product path
fails loudly when its CUDA library is missing instead of falling back here.

Parity pin: the oracle is checked against golden vectors produced by running
the reference itself (`tests/golden/make_golden.py`, fixtures in
`tests/golden/*.npz`; test `tests/test_oracle_golden.py`).

Data model (differs from the reference's classes on purpose): a prognostic
state is one complex128 array of shape (3, R+1, R+1) holding
(phi_prime, zeta, delta) in that order, dense triangular layout [r, s] with
structural zeros for s < r (spharm.py:6-10).  Grids are (n_lon, n_lat)
float64, longitude-major, latitudes ascending in mu (spharm.py:3-5).

Arithmetic is the reference's: dense (R+1, R+1, J) tables, pocketfft via
numpy for the longitude transforms, batched matmul for the Legendre sums, so
timing this module is a fair stand-in for timing the reference's CPU path.
"""

from __future__ import annotations

import math

import numpy as np

PHI, ZETA, DELTA = 0, 1, 2


# ----------------------------------------------------------------------------
# Gaussian grid  (spharm.py:40-138)
# ----------------------------------------------------------------------------

def fast_size(n: int) -> int:
    """Smallest m >= n with prime factors in {2,3,5} (spharm.py:40-49)."""
    m = n
    while True:
        k = m
        for p in (2, 3, 5):
            while k % p == 0:
                k //= p
        if k == 1:
            return m
        m += 1


def gauss_nodes(n: int, tol: float = 1e-14, max_iter: int = 100):
    """Gauss-Legendre nodes/weights, ascending and symmetrised.

    Newton on the three-term Legendre recurrence from the guesses
    cos(pi (k - 1/4) / (n + 1/2)) (spharm.py:52-86).  The operation order
    matches the reference so the result is bitwise identical.
    """
    if n < 1:
        raise ValueError(f"need at least one node, got {n}")
    x = np.cos(np.pi * (np.arange(1, n + 1) - 0.25) / (n + 0.5))
    ok = np.zeros(n, dtype=bool)
    deriv = np.empty_like(x)
    for _ in range(max_iter):
        pm1 = np.ones_like(x)
        p = x.copy()
        for k in range(2, n + 1):
            pm1, p = p, ((2 * k - 1) * x * p - (k - 1) * pm1) / k
        deriv = n * (x * p - pm1) / (x * x - 1.0)
        step = p / deriv
        x -= step
        ok = np.abs(step) <= tol
        if ok.all():
            break
    if not ok.all():
        raise RuntimeError(f"Gauss-Legendre root search failed to converge for n={n}")
    w = 2.0 / ((1.0 - x * x) * deriv * deriv)
    idx = np.argsort(x)
    x, w = x[idx], w[idx]
    return 0.5 * (x - x[::-1]), 0.5 * (w + w[::-1])


def default_shape(R: int):
    """(n_lon, n_lat) dealiased grid for truncation R (spharm.py:130-138)."""
    return fast_size(3 * R + 1), -(-(3 * R + 1) // 2)


# ----------------------------------------------------------------------------
# Legendre tables  (spharm.py:141-179)
# ----------------------------------------------------------------------------

def legendre_pbar(R: int, mu: np.ndarray, degree_max: int | None = None) -> np.ndarray:
    """P[r, s, j] = orthonormal Pbar_s^r(mu_j) for s <= degree_max.

    Sectoral seed Pbar_r^r, first step mu sqrt(2r+3) Pbar_r^r, then the
    upward three-term recurrence in s (spharm.py:153-169).
    """
    smax = R + 1 if degree_max is None else degree_max
    J = mu.size
    P = np.zeros((R + 1, smax + 1, J))
    cosphi = np.sqrt(1.0 - mu * mu)
    seed = np.full(J, 1.0 / np.sqrt(2.0))
    for r in range(R + 1):
        P[r, r] = seed
        if r + 1 <= smax:
            P[r, r + 1] = mu * np.sqrt(2.0 * r + 3.0) * seed
        for s in range(r + 2, smax + 1):
            s2, r2 = s * s, r * r
            a = np.sqrt((4.0 * s2 - 1.0) / (s2 - r2))
            b = np.sqrt((2.0 * s + 1.0) * (s - 1.0 - r) * (s - 1.0 + r)
                        / ((2.0 * s - 3.0) * (s2 - r2)))
            P[r, s] = a * mu * P[r, s - 1] - b * P[r, s - 2]
        seed = seed * cosphi * np.sqrt((2.0 * r + 3.0) / (2.0 * r + 2.0))
    return P


def legendre_h(R: int, P: np.ndarray) -> np.ndarray:
    """H = (1 - mu^2) dPbar/dmu from P at s -+ 1 (spharm.py:171-178)."""
    H = np.zeros((R + 1, R + 1, P.shape[-1]))
    for r in range(R + 1):
        for s in range(r, R + 1):
            up = np.sqrt(((s + 1.0) ** 2 - r * r) / (4.0 * (s + 1.0) ** 2 - 1.0))
            H[r, s] = -s * up * P[r, s + 1]
            if s > r:
                dn = np.sqrt((s * s - r * r) / (4.0 * s * s - 1.0))
                H[r, s] += (s + 1.0) * dn * P[r, s - 1]
    return H


# ----------------------------------------------------------------------------
# Spectral operators  (spharm.py:303-349)
# ----------------------------------------------------------------------------

def lap_eigs(R: int, a: float) -> np.ndarray:
    """-s(s+1)/a^2 per total wavenumber s (spharm.py:307-310)."""
    s = np.arange(R + 1, dtype=float)
    return -s * (s + 1.0) / (a * a)


def lap(c: np.ndarray, a: float) -> np.ndarray:
    """spharm.py:313-317."""
    if a <= 0:
        raise ValueError("radius must be positive")
    return c * lap_eigs(c.shape[-1] - 1, a)


def invlap(c: np.ndarray, a: float) -> np.ndarray:
    """Inverse Laplacian, s=0 gauged to zero (spharm.py:320-328)."""
    if a <= 0:
        raise ValueError("radius must be positive")
    ev = lap_eigs(c.shape[-1] - 1, a)
    ev[0] = 1.0
    out = c / ev
    out[..., 0] = 0.0
    return out


def trunc(c: np.ndarray, Rc: int) -> np.ndarray:
    """spharm.py:331-336."""
    if Rc > c.shape[-1] - 1:
        raise ValueError("cannot truncate to a larger truncation")
    return c[..., : Rc + 1, : Rc + 1].copy()


def pad(c: np.ndarray, Rf: int) -> np.ndarray:
    """spharm.py:339-349."""
    Rin = c.shape[-1] - 1
    if Rf < Rin:
        raise ValueError("cannot pad to a smaller truncation")
    out = np.zeros(c.shape[:-2] + (Rf + 1, Rf + 1), dtype=c.dtype)
    out[..., : Rin + 1, : Rin + 1] = c
    return out


# ----------------------------------------------------------------------------
# Transform plan  (spharm.py:182-300)
# ----------------------------------------------------------------------------

class OraclePlan:
    """Dense-table SH transform at truncation R on an (n_lon, n_lat) grid."""

    def __init__(self, R: int, n_lon: int, n_lat: int):
        if R < 0:
            raise ValueError("truncation must be non-negative")
        if n_lon < 2 * R + 1:
            raise ValueError("n_lon cannot carry the zonal wavenumbers")
        self.R, self.I, self.J = R, n_lon, n_lat
        self.mu, self.w = gauss_nodes(n_lat)
        Pfull = legendre_pbar(R, self.mu)
        self.P = Pfull[:, : R + 1, :]
        self.H = legendre_h(R, Pfull)
        wc2 = self.w / (1.0 - self.mu ** 2)
        self.Pw = self.P * self.w             # spharm.py:203
        self.Pwc2 = self.P * wc2              # spharm.py:204
        self.Hwc2 = self.H * wc2              # spharm.py:205
        self.ir = 1j * np.arange(R + 1)[:, None]

    # -- longitude halves (spharm.py:210-222)
    def to_fourier(self, g: np.ndarray) -> np.ndarray:
        if g.shape != (self.I, self.J):
            raise ValueError(f"field shape {g.shape} does not match grid ({self.I}, {self.J})")
        return np.fft.rfft(g, axis=0)[: self.R + 1] / self.I

    def to_grid(self, f: np.ndarray) -> np.ndarray:
        spec = np.zeros((self.I // 2 + 1, self.J), dtype=complex)
        spec[: self.R + 1] = f
        return np.fft.irfft(spec * self.I, n=self.I, axis=0)

    # -- Legendre contractions (spharm.py:224-250)
    @staticmethod
    def _ana(table: np.ndarray, f: np.ndarray) -> np.ndarray:
        y = table @ np.stack([f.real, f.imag], axis=-1)
        return y[..., 0] + 1j * y[..., 1]

    def _syn(self, table: np.ndarray, c: np.ndarray) -> np.ndarray:
        Rin = c.shape[-1] - 1
        if Rin > self.R:
            raise ValueError("coefficients exceed plan truncation")
        if Rin < self.R:
            c = pad(c, self.R)
        y = np.stack([c.real, c.imag], axis=1) @ table
        return y[:, 0, :] + 1j * y[:, 1, :]

    # -- public transforms (spharm.py:254-300)
    def analyze(self, g: np.ndarray) -> np.ndarray:
        return self._ana(self.Pw, self.to_fourier(g))

    def synthesize(self, c: np.ndarray) -> np.ndarray:
        return self.to_grid(self._syn(self.P, c))

    def synth_uv(self, psi: np.ndarray, chi: np.ndarray):
        """U = i r P chi - H psi, V = i r P psi + H chi (spharm.py:262-279)."""
        fu = self.ir * self._syn(self.P, chi) - self._syn(self.H, psi)
        fv = self.ir * self._syn(self.P, psi) + self._syn(self.H, chi)
        return self.to_grid(fu), self.to_grid(fv)

    def anal_divcurl(self, gu: np.ndarray, gv: np.ndarray):
        """div/curl of a cos-weighted vector field (spharm.py:281-300)."""
        fa, fb = self.to_fourier(gu), self.to_fourier(gv)
        div = self._ana(self.Pwc2, self.ir * fa) - self._ana(self.Hwc2, fb)
        curl = self._ana(self.Pwc2, self.ir * fb) + self._ana(self.Hwc2, fa)
        return div, curl


# ----------------------------------------------------------------------------
# Shallow-water operators  (swe.py:20-288, implicit.py:31-49)
# ----------------------------------------------------------------------------

class OracleParams:
    """swe.py:20-41; phi_bar = g * h_bar."""

    def __init__(self, radius=6.37122e6, omega=7.292e-5, gravity=9.80616, nu=1.0e5, h_bar=1.0e4):
        if radius <= 0 or gravity <= 0 or h_bar <= 0:
            raise ValueError("radius, gravity and h_bar must be positive")
        if nu < 0:
            raise ValueError("diffusion coefficient must be non-negative")
        self.radius, self.omega, self.gravity, self.nu, self.h_bar = radius, omega, gravity, nu, h_bar
        self.phi_bar = gravity * h_bar


class OracleRHS:
    """Split right-hand sides F_I (implicit) and F_E (explicit), swe.py:157-288."""

    def __init__(self, plan: OraclePlan, params: OracleParams, nonlinear: bool = True):
        self.plan, self.prm, self.nonlinear = plan, params, nonlinear
        self.lam = lap_eigs(plan.R, params.radius)
        self.f_grid = 2.0 * params.omega * plan.mu[None, :]
        self.c2o = 2.0 * params.omega / params.radius
        self.inv_c2 = 1.0 / (1.0 - plan.mu[None, :] ** 2)
        self.n_solve = self.n_fi = self.n_fe = 0

    def velocities(self, st):
        """Cos-weighted winds via psi, chi (swe.py:184-190)."""
        a = self.prm.radius
        psi, chi = invlap(st[ZETA], a), invlap(st[DELTA], a)
        u, v = self.plan.synth_uv(psi, chi)
        return u * (1.0 / a), v * (1.0 / a)

    def divcurl(self, gu, gv):
        d, c = self.plan.anal_divcurl(gu, gv)
        s = 1.0 / self.prm.radius
        return d * s, c * s

    def l_g(self, st):
        """swe.py:206-217."""
        nl = self.prm.nu * self.lam
        return np.stack([
            -self.prm.phi_bar * st[DELTA] + nl * st[PHI],
            nl * st[ZETA],
            -self.lam * st[PHI] + nl * st[DELTA],
        ])

    def eval_fi(self, st):
        """swe.py:246-249."""
        self.n_fi += 1
        return self.l_g(st)

    def eval_fe(self, st):
        """Fused Coriolis + advection terms, swe.py:251-279."""
        self.n_fe += 1
        p = self.plan
        u, v = self.velocities(st)
        zg = p.synthesize(st[ZETA])
        dg = p.synthesize(st[DELTA])
        out = np.zeros_like(st)
        out[ZETA] = p.analyze(-self.f_grid * dg - self.c2o * v)
        out[DELTA] = p.analyze(self.f_grid * zg - self.c2o * u)
        if not self.nonlinear:
            return out
        pg = p.synthesize(st[PHI])
        div_phi, _ = self.divcurl(pg * u, pg * v)
        div_z, curl_z = self.divcurl(zg * u, zg * v)
        ke = 0.5 * (u * u + v * v) * self.inv_c2
        lap_ke = lap(p.analyze(ke), self.prm.radius)
        out[PHI] = out[PHI] - div_phi
        out[ZETA] = out[ZETA] - div_z
        out[DELTA] = out[DELTA] + (curl_z - lap_ke)
        return out

    def solve(self, b, beta: float):
        """(I - beta F_I) theta = b, mode by mode (implicit.py:31-49)."""
        if beta < 0:
            raise ValueError("implicit step must be non-negative")
        self.n_solve += 1
        lam, nu, pb = self.lam, self.prm.nu, self.prm.phi_bar
        d = 1.0 - beta * nu * lam
        det = d * d - beta * beta * lam * pb
        if np.any(det <= 0.0):
            raise RuntimeError("implicit system is singular; invalid model parameters")
        return np.stack([
            (d * b[PHI] - beta * pb * b[DELTA]) / det,
            b[ZETA] / d,
            (d * b[DELTA] - beta * lam * b[PHI]) / det,
        ])


# ----------------------------------------------------------------------------
# Collocation tables  (sdc.py:24-134; mlsdc.py:41-56)
# ----------------------------------------------------------------------------

def lobatto(n: int) -> np.ndarray:
    """sdc.py:24-39."""
    if n == 2:
        return np.array([0.0, 1.0])
    if n == 3:
        return np.array([0.0, 0.5, 1.0])
    if n == 5:
        c = math.sqrt(3.0 / 7.0)
        return np.array([0.0, 0.5 * (1.0 - c), 0.5, 0.5 * (1.0 + c), 1.0])
    raise ValueError(f"unsupported node count {n}")


def q_matrix(t: np.ndarray) -> np.ndarray:
    """Integrals of the Lagrange basis from t_0 to t_m (sdc.py:42-62)."""
    n = t.size
    q = np.zeros((n, n))
    for j in range(n):
        others = np.delete(t, j)
        poly = np.polynomial.Polynomial.fromroots(others) / np.prod(t[j] - others)
        anti = poly.integ()
        q[:, j] = anti(t) - anti(t[0])
    return q


def _doolittle_upper(a: np.ndarray) -> np.ndarray:
    """No-pivot LU, returns U; raises on a zero pivot (sdc.py:65-79)."""
    n = a.shape[0]
    u = a.astype(float).copy()
    for k in range(n - 1):
        if u[k, k] == 0.0:
            raise RuntimeError("zero pivot in LU factorization of the weight block")
        for i in range(k + 1, n):
            l = u[i, k] / u[k, k]
            u[i, k:] -= l * u[k, k:]
            u[i, k] = 0.0
    if u[n - 1, n - 1] == 0.0:
        raise RuntimeError("zero pivot in LU factorization of the weight block")
    return u


def qdelta_i(q: np.ndarray) -> np.ndarray:
    """LU-trick implicit weights (sdc.py:82-95)."""
    n = q.shape[0]
    out = np.zeros((n, n))
    out[1:, 1:] = _doolittle_upper(q[1:, 1:].T).T
    return out


def qdelta_e(t: np.ndarray) -> np.ndarray:
    """Forward-Euler weights (sdc.py:98-109)."""
    n = t.size
    out = np.zeros((n, n))
    h = np.diff(t)
    for m in range(1, n):
        out[m, :m] = h[:m]
    return out


class OracleTables:
    def __init__(self, n_nodes: int):
        self.t = lobatto(n_nodes)
        self.q = q_matrix(self.t)
        self.qi = qdelta_i(self.q)
        self.qe = qdelta_e(self.t)
        self.n = n_nodes


def lagrange_transfer(t_from: np.ndarray, t_to: np.ndarray) -> np.ndarray:
    """Row i = Lagrange basis of t_from evaluated at t_to[i] (mlsdc.py:41-56)."""
    out = np.empty((t_to.size, t_from.size))
    for j, tj in enumerate(t_from):
        others = np.delete(t_from, j)
        den = np.prod(tj - others)
        for i, ti in enumerate(t_to):
            out[i, j] = np.prod(ti - others) / den
    return out


# ----------------------------------------------------------------------------
# Sweeps  (sdc.py:156-253)
# ----------------------------------------------------------------------------

def weighted_sum(weights, states):
    """Sum of w_k * x_k skipping exactly-zero weights (sdc.py:211-220)."""
    acc = None
    for wk, xk in zip(weights, states):
        if wk == 0.0:
            continue
        acc = wk * xk if acc is None else acc + wk * xk
    return np.zeros_like(states[0]) if acc is None else acc


class Nodes:
    """Node states and cached tendencies (sdc.py:137-153); lists of arrays."""

    def __init__(self, theta, fi, fe):
        self.theta, self.fi, self.fe = theta, fi, fe

    @classmethod
    def start(cls, st, rhs: OracleRHS, n: int):
        """sdc.py:156-170."""
        fi, fe = rhs.eval_fi(st), rhs.eval_fe(st)
        return cls([st.copy() for _ in range(n)], [fi.copy() for _ in range(n)],
                   [fe.copy() for _ in range(n)])


def sweep(nd: Nodes, tb: OracleTables, dt: float, rhs: OracleRHS, tau=None):
    """One IMEX SDC sweep over nodes 1..M in place (sdc.py:173-208)."""
    n = len(nd.theta)
    f_old = [nd.fi[j] + nd.fe[j] for j in range(n)]
    quad = [None] + [dt * weighted_sum(tb.q[m], f_old) for m in range(1, n)]
    fi_old, fe_old = list(nd.fi), list(nd.fe)
    for m in range(1, n):
        b = nd.theta[0] + quad[m]
        for j in range(1, m):
            b = b + (dt * tb.qe[m, j]) * (nd.fe[j] - fe_old[j])
            b = b + (dt * tb.qi[m, j]) * (nd.fi[j] - fi_old[j])
        b = b + (-dt * tb.qi[m, m]) * fi_old[m]
        if tau is not None:
            b = b + tau[m]
        th = rhs.solve(b, dt * tb.qi[m, m])
        nd.theta[m] = th
        nd.fi[m] = rhs.eval_fi(th)
        nd.fe[m] = rhs.eval_fe(th)
    return nd


def sdc_step(st, dt: float, n_sweeps: int, tb: OracleTables, rhs: OracleRHS):
    """sdc.py:236-253."""
    if n_sweeps < 1:
        raise ValueError("at least one sweep is required")
    nd = Nodes.start(st, rhs, tb.n)
    for _ in range(n_sweeps):
        sweep(nd, tb, dt, rhs)
    return nd.theta[-1]


# ----------------------------------------------------------------------------
# Two-level MLSDC  (mlsdc.py:59-254)
# ----------------------------------------------------------------------------

class OracleLevel:
    def __init__(self, R: int, n_nodes: int, params: OracleParams, grid_shape=None, nonlinear=True):
        I, J = grid_shape if grid_shape else default_shape(R)
        self.plan = OraclePlan(R, I, J)
        self.tb = OracleTables(n_nodes)
        self.rhs = OracleRHS(self.plan, params, nonlinear)
        self.R = R


class OracleHierarchy:
    """Fine/coarse levels plus time transfer (mlsdc.py:59-95, 139-181)."""

    def __init__(self, fine: OracleLevel, coarse: OracleLevel):
        if coarse.tb.n > fine.tb.n:
            raise ValueError("coarse level cannot have more nodes than fine")
        if coarse.R > fine.R:
            raise ValueError("coarse truncation cannot exceed fine truncation")
        self.fine, self.coarse = fine, coarse
        self.pi_fc = lagrange_transfer(fine.tb.t, coarse.tb.t)
        self.pi_cf = lagrange_transfer(coarse.tb.t, fine.tb.t)

    def restrict(self, states):
        """mlsdc.py:83-88."""
        return [trunc(weighted_sum(row, states), self.coarse.R) for row in self.pi_fc]

    def interpolate(self, states):
        """mlsdc.py:90-95."""
        up = [pad(s, self.fine.R) for s in states]
        return [weighted_sum(row, up) for row in self.pi_cf]


def fas_tau(h: OracleHierarchy, ndf: Nodes, ndc: Nodes, dt: float):
    """tau_c = R(dt Q_f F_f) - dt Q_c F_c (mlsdc.py:98-124)."""
    ff = [ndf.fi[j] + ndf.fe[j] for j in range(len(ndf.theta))]
    intf = [dt * weighted_sum(row, ff) for row in h.fine.tb.q]
    rest = h.restrict(intf)
    fc = [ndc.fi[j] + ndc.fe[j] for j in range(len(ndc.theta))]
    return [rest[m] - dt * weighted_sum(h.coarse.tb.q[m], fc) for m in range(len(ndc.theta))]


def mlsdc_start(st, h: OracleHierarchy):
    """mlsdc.py:184-199."""
    ndf = Nodes.start(st, h.fine.rhs, h.fine.tb.n)
    c0 = trunc(st, h.coarse.R)
    fi, fe = h.coarse.rhs.eval_fi(c0), h.coarse.rhs.eval_fe(c0)
    n = h.coarse.tb.n
    ndc = Nodes([c0.copy() for _ in range(n)], [fi.copy() for _ in range(n)],
                [fe.copy() for _ in range(n)])
    return ndf, ndc


def mlsdc_iter(ndf: Nodes, ndc: Nodes, h: OracleHierarchy, dt: float, coarse_sweeps: int = 1):
    """V-cycle A-D (mlsdc.py:202-239).  coarse_sweeps > 1 repeats the
    coarse FAS sweep with the same tau (composed from
    mlsdc.py:127-136)."""
    fine, coarse = h.fine, h.coarse
    sweep(ndf, fine.tb, dt, fine.rhs)
    rest = h.restrict(ndf.theta)
    for m in range(1, coarse.tb.n):
        ndc.theta[m] = rest[m]
        ndc.fi[m] = coarse.rhs.eval_fi(rest[m])
        ndc.fe[m] = coarse.rhs.eval_fe(rest[m])
    s_th = [x.copy() for x in ndc.theta]
    s_fi = [x.copy() for x in ndc.fi]
    s_fe = [x.copy() for x in ndc.fe]
    tau = fas_tau(h, ndf, ndc, dt)
    for _ in range(coarse_sweeps):
        sweep(ndc, coarse.tb, dt, coarse.rhs, tau)
    nc = coarse.tb.n
    d_th = h.interpolate([ndc.theta[m] - s_th[m] for m in range(nc)])
    d_fi = h.interpolate([ndc.fi[m] - s_fi[m] for m in range(nc)])
    d_fe = h.interpolate([ndc.fe[m] - s_fe[m] for m in range(nc)])
    for m in range(1, fine.tb.n):
        ndf.theta[m] = ndf.theta[m] + d_th[m]
        ndf.fi[m] = ndf.fi[m] + d_fi[m]
        ndf.fe[m] = ndf.fe[m] + d_fe[m]
    return ndf


def mlsdc_step(st, dt: float, n_iter: int, h: OracleHierarchy, coarse_sweeps: int = 1):
    """mlsdc.py:242-254."""
    if n_iter < 1:
        raise ValueError("at least one iteration is required")
    ndf, ndc = mlsdc_start(st, h)
    for _ in range(n_iter):
        mlsdc_iter(ndf, ndc, h, dt, coarse_sweeps)
    return ndf.theta[-1]
