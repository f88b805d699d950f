"""Streaming per-r CPU oracle for large truncations -- TEST INFRASTRUCTURE ONLY.

The reference's TransformPlan (spharm.py:182-206) stores five dense
(R+1, R+1, J) tables; at T1279 on 1920 latitudes that is 126 GB, so neither
the reference nor the dense restatement in `swsdc_oracle.py` can be built
there.  This module restates the same algorithm with the
tables generated block by block over the zonal wavenumber r and consumed as
soon as they are made:

* the Legendre recurrence of spharm.py:141-169 with the reference's exact
  per-element arithmetic (same operations in the same order, vectorised over
  the r of a block instead of looping over r), so every table entry is
  bitwise equal to the dense one;
* H from P at s -+ 1 as in spharm.py:171-178 (also bitwise equal);
* the weighted tables of spharm.py:201-205 (P*w, P*w/(1-mu^2), H*w/(1-mu^2));
* the contractions of spharm.py:224-250 as per-r matmuls over s >= r0 (the
  block's first r), which only drops structural zeros -- results differ from
  the dense plan by summation order (~1e-16 relative);
* the longitude transforms of spharm.py:210-222 (numpy pocketfft, unchanged).

`StreamRHS.eval_fe` evaluates swe.py:251-279 with all 18 contractions of one
evaluation grouped into two table passes (7 synthesis contractions, then 11
analysis contractions), which is the only reason it is a separate class.

Only `tests/` and the golden generators import this module.  It is validated
against the reference itself at T255 and T639 (`tests/golden/make_golden_large.py`,
which writes the validation deviations into the fixture it produces).
"""

from __future__ import annotations

import numpy as np

from swsdc_oracle import (DELTA, PHI, ZETA, OracleHierarchy, OracleParams, OracleRHS,
                          OracleTables, default_shape, gauss_nodes, lap, pad)


def _sectoral_seeds(R: int, mu: np.ndarray) -> np.ndarray:
    """Pbar_r^r(mu_j) for r = 0..R+1, the sequential seed chain of
    spharm.py:153-169 (seed_{r+1} = seed_r * cos(phi) * sqrt((2r+3)/(2r+2)))."""
    cosphi = np.sqrt(1.0 - mu * mu)
    out = np.empty((R + 2, mu.size))
    seed = np.full(mu.size, 1.0 / np.sqrt(2.0))
    for r in range(R + 2):
        out[r] = seed
        seed = seed * cosphi * np.sqrt((2.0 * r + 3.0) / (2.0 * r + 2.0))
    return out


class StreamPlan:
    """SH transform at truncation R on an (n_lon, n_lat) grid whose Legendre
    tables are generated per block of zonal wavenumbers (spharm.py:182-300)."""

    def __init__(self, R: int, n_lon: int, n_lat: int, block_bytes: float = 3.0e8):
        if R < 0:
            raise ValueError("truncation must be non-negative")
        if n_lon < 2 * R + 1:
            raise ValueError("n_lon cannot carry the zonal wavenumbers")
        self.R, self.I, self.J = R, n_lon, n_lat
        self.mu, self.w = gauss_nodes(n_lat)
        self.wc2 = self.w / (1.0 - self.mu ** 2)
        self.seeds = _sectoral_seeds(R, self.mu)
        self.ir = 1j * np.arange(R + 1)[:, None]
        per_row = (R + 2) * n_lat * 8.0
        self.rb = int(max(1, min(R + 1, block_bytes // per_row)))

    # -- tables of one r-block  (spharm.py:141-179) ---------------------------
    def _p_block(self, r0: int, r1: int) -> np.ndarray:
        """P[r - r0, s - r0, j] for r0 <= r < r1 and r0 <= s <= R+1."""
        R, mu = self.R, self.mu
        smax = R + 1
        nb, ns = r1 - r0, smax + 1 - r0
        P = np.zeros((nb, ns, mu.size))
        for i in range(nb):
            r = r0 + i
            P[i, r - r0] = self.seeds[r]
            if r + 1 <= smax:
                P[i, r + 1 - r0] = mu * np.sqrt(2.0 * r + 3.0) * self.seeds[r]
        rr = np.arange(r0, r1)
        for s in range(r0 + 2, smax + 1):
            k = min(nb, s - 2 - r0 + 1)          # rows with r <= s - 2
            r = rr[:k]
            s2, r2 = s * s, r * r
            a = np.sqrt((4.0 * s2 - 1.0) / (s2 - r2))
            b = np.sqrt((2.0 * s + 1.0) * (s - 1.0 - r) * (s - 1.0 + r)
                        / ((2.0 * s - 3.0) * (s2 - r2)))
            si = s - r0
            P[:k, si] = (a[:, None] * mu) * P[:k, si - 1] - b[:, None] * P[:k, si - 2]
        return P

    def _h_block(self, r0: int, r1: int, P: np.ndarray) -> np.ndarray:
        """H[r - r0, s - r0, j] for s <= R (spharm.py:171-178)."""
        R = self.R
        H = np.zeros((r1 - r0, R + 1 - r0, self.J))
        for i in range(r1 - r0):
            r = r0 + i
            s = np.arange(r, R + 1)
            up = np.sqrt(((s + 1.0) ** 2 - r * r) / (4.0 * (s + 1.0) ** 2 - 1.0))
            si = s - r0
            H[i, si] = ((-s) * up)[:, None] * P[i, si + 1]
            if R > r:
                s = s[1:]
                dn = np.sqrt((s * s - r * r) / (4.0 * s * s - 1.0))
                H[i, s - r0] += ((s + 1.0) * dn)[:, None] * P[i, s - 1 - r0]
        return H

    def blocks(self, need_h: bool):
        """Yield (r0, r1, P, H) with P, H restricted to s <= R."""
        for r0 in range(0, self.R + 1, self.rb):
            r1 = min(self.R + 1, r0 + self.rb)
            Pf = self._p_block(r0, r1)
            H = self._h_block(r0, r1, Pf) if need_h else None
            yield r0, r1, Pf[:, : self.R + 1 - r0], H

    # -- longitude halves (spharm.py:210-222) ---------------------------------
    def to_fourier(self, g: np.ndarray) -> np.ndarray:
        if g.shape != (self.I, self.J):
            raise ValueError(f"field shape {g.shape} does not match grid ({self.I}, {self.J})")
        return np.fft.rfft(g, axis=0)[: self.R + 1] / self.I

    def to_grid(self, f: np.ndarray) -> np.ndarray:
        spec = np.zeros((self.I // 2 + 1, self.J), dtype=complex)
        spec[: self.R + 1] = f
        return np.fft.irfft(spec * self.I, n=self.I, axis=0)

    # -- batched contractions (spharm.py:224-250) -----------------------------
    def _coeff(self, c: np.ndarray) -> np.ndarray:
        Rin = c.shape[-1] - 1
        if Rin > self.R:
            raise ValueError("coefficients exceed plan truncation")
        return pad(c, self.R) if Rin < self.R else c

    def contract(self, syn=(), ana=()):
        """syn: list of (table, coeffs) with table in {'P', 'H'};
        ana: list of (table, fourier) with table in {'Pw', 'Pwc2', 'Hwc2'}.
        Returns ([Fourier rows per syn job], [coefficients per ana job])."""
        R, J = self.R, self.J
        syn = [(t, self._coeff(c)) for t, c in syn]
        need_h = any(t == "H" for t, _ in syn) or any(t == "Hwc2" for t, _ in ana)
        fo = [np.zeros((R + 1, J), dtype=complex) for _ in syn]
        co = [np.zeros((R + 1, R + 1), dtype=complex) for _ in ana]
        fr = [np.stack([f.real, f.imag], axis=-1) for _, f in ana]
        for r0, r1, P, H in self.blocks(need_h):
            tabs = {"P": P, "H": H}
            if any(t == "Pw" for t, _ in ana):
                tabs["Pw"] = P * self.w
            if any(t == "Pwc2" for t, _ in ana):
                tabs["Pwc2"] = P * self.wc2
            if any(t == "Hwc2" for t, _ in ana):
                tabs["Hwc2"] = H * self.wc2
            for k, (t, c) in enumerate(syn):
                cb = c[r0:r1, r0:]
                y = np.stack([cb.real, cb.imag], axis=1) @ tabs[t]
                fo[k][r0:r1] = y[:, 0, :] + 1j * y[:, 1, :]
            for k, (t, _) in enumerate(ana):
                y = tabs[t] @ fr[k][r0:r1]
                co[k][r0:r1, r0:] = y[..., 0] + 1j * y[..., 1]
        return fo, co

    # -- public transforms (spharm.py:254-300) --------------------------------
    def analyze(self, g: np.ndarray) -> np.ndarray:
        return self.contract(ana=[("Pw", self.to_fourier(g))])[1][0]

    def synthesize(self, c: np.ndarray) -> np.ndarray:
        return self.to_grid(self.contract(syn=[("P", c)])[0][0])

    def synth_uv(self, psi: np.ndarray, chi: np.ndarray):
        """U = i r P chi - H psi, V = i r P psi + H chi (spharm.py:262-279)."""
        (pc, hp, pp, hc), _ = self.contract(syn=[("P", chi), ("H", psi), ("P", psi), ("H", chi)])
        return self.to_grid(self.ir * pc - hp), self.to_grid(self.ir * pp + hc)

    def anal_divcurl(self, gu: np.ndarray, gv: np.ndarray):
        """spharm.py:281-300."""
        fa, fb = self.to_fourier(gu), self.to_fourier(gv)
        _, (d1, d2, c1, c2) = self.contract(ana=[("Pwc2", self.ir * fa), ("Hwc2", fb),
                                                 ("Pwc2", self.ir * fb), ("Hwc2", fa)])
        return d1 - d2, c1 + c2


class StreamRHS(OracleRHS):
    """OracleRHS over a StreamPlan; eval_fe (swe.py:251-279) batches its 18
    contractions into one synthesis pass and one analysis pass."""

    def eval_fe(self, st):
        self.n_fe += 1
        p, a = self.plan, self.prm.radius
        from swsdc_oracle import invlap
        psi, chi = invlap(st[ZETA], a), invlap(st[DELTA], a)
        syn = [("P", chi), ("H", psi), ("P", psi), ("H", chi), ("P", st[ZETA]), ("P", st[DELTA])]
        if self.nonlinear:
            syn.append(("P", st[PHI]))
        fo, _ = p.contract(syn=syn)
        u = p.to_grid(p.ir * fo[0] - fo[1]) * (1.0 / a)
        v = p.to_grid(p.ir * fo[2] + fo[3]) * (1.0 / a)
        zg, dg = p.to_grid(fo[4]), p.to_grid(fo[5])
        ana = [("Pw", p.to_fourier(-self.f_grid * dg - self.c2o * v)),
               ("Pw", p.to_fourier(self.f_grid * zg - self.c2o * u))]
        if self.nonlinear:
            pg = p.to_grid(fo[6])
            ke = 0.5 * (u * u + v * v) * self.inv_c2
            for gu, gv in ((pg * u, pg * v), (zg * u, zg * v)):
                fa, fb = p.to_fourier(gu), p.to_fourier(gv)
                ana += [("Pwc2", p.ir * fa), ("Hwc2", fb), ("Pwc2", p.ir * fb), ("Hwc2", fa)]
            ana.append(("Pw", p.to_fourier(ke)))
        _, co = p.contract(ana=ana)
        out = np.zeros_like(st)
        out[ZETA], out[DELTA] = co[0], co[1]
        if not self.nonlinear:
            return out
        s = 1.0 / a
        div_phi = (co[2] - co[3]) * s
        div_z, curl_z = (co[6] - co[7]) * s, (co[8] + co[9]) * s
        lap_ke = lap(co[10], a)
        out[PHI] = out[PHI] - div_phi
        out[ZETA] = out[ZETA] - div_z
        out[DELTA] = out[DELTA] + (curl_z - lap_ke)
        return out


class StreamLevel:
    """OracleLevel with a StreamPlan (duck-typed for OracleHierarchy)."""

    def __init__(self, R: int, n_nodes: int, params: OracleParams, grid_shape=None,
                 nonlinear=True, block_bytes: float = 3.0e8):
        I, J = grid_shape if grid_shape else default_shape(R)
        self.plan = StreamPlan(R, I, J, block_bytes)
        self.tb = OracleTables(n_nodes)
        self.rhs = StreamRHS(self.plan, params, nonlinear)
        self.R = R


__all__ = ["StreamPlan", "StreamRHS", "StreamLevel", "OracleHierarchy"]
