"""Which r = 0 Legendre analysis is closer to exact arithmetic at T1279: the
reference's recurrence (spharm.py:160-168, s steps of rounding) or the GPU's
scaled recurrence restarted from exact checkpoints every 32 degrees?  Exact =
the reference recurrence in long double (64-bit mantissa).  Input: the zonal
mean of a kinetic-energy-like positive field (smooth, large mean), whose
high-degree coefficients are the ill-conditioned ones; errors are reported
times s(s+1) (the Laplacian of the F_E delta tendency, swe.py:273)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import swsdc_oracle as orc

R, J = int(sys.argv[1]) if len(sys.argv) > 1 else 1279, None
J = {255: 384, 639: 960, 1279: 1920}[R]
mu, w = orc.gauss_nodes(J)
rng = np.random.default_rng(3)
# smooth positive profile: 1 + sum of a few low-degree Legendre-like modes squared
u = sum(rng.normal() * np.cos(k * np.arccos(mu)) / (k + 1) ** 2 for k in range(40))
F = 0.5 * (u * u + 0.3) / (1 - mu * mu) * (1 - mu * mu)  # positive, large mean

def pref(dtype):
    m = mu.astype(dtype)
    P = np.zeros((R + 2, J), dtype=dtype)
    P[0] = dtype(1.0) / np.sqrt(dtype(2.0))
    P[1] = m * np.sqrt(dtype(3.0)) * P[0]
    for s in range(2, R + 2):
        a = np.sqrt(dtype(4 * s * s - 1) / dtype(s * s))
        b = np.sqrt(dtype(2 * s + 1) * dtype(s - 1) * dtype(s - 1) / (dtype(2 * s - 3) * dtype(s * s)))
        P[s] = a * m * P[s - 1] - b * P[s - 2]
    return P[: R + 1]

Pd, Pl = pref(np.float64), pref(np.longdouble)
# GPU-like: scaled recurrence between exact (double reference) checkpoints
K = 32
a = np.zeros(R + 2); b = np.zeros(R + 2)
a[1] = np.sqrt(3.0)
s = np.arange(2, R + 2)
a[2:] = np.sqrt((4.0 * s * s - 1.0) / (s * s).astype(float))
b[2:] = np.sqrt((2.0 * s + 1.0) * (s - 1.0) * (s - 1.0) / ((2.0 * s - 3.0) * (s * s).astype(float)))
beta = np.zeros(R + 2); beta[2:] = b[2:] / (a[2:] * a[1:-1])
g = np.ones(R + 2)
for k in range(1, R + 2):
    g[k] = 1.0 if k % K == 0 else g[k - 1] * a[k]
Pg = Pd.copy()
ml = mu.astype(np.longdouble)
for k0 in range(0, R + 1, K):
    qa = Pd[k0]
    if k0 + 1 > R: break
    qb = Pd[k0 + 1] / a[k0 + 1]
    Pg[k0 + 1] = qb * g[k0 + 1]
    for k in range(k0 + 2, min(k0 + K, R + 1)):
        qn = (ml * qb + ((-beta[k]) * qa)).astype(np.float64)
        Pg[k] = qn * g[k]
        qa, qb = qb, qn
cl = (Pl * (w * F).astype(np.longdouble)).sum(axis=1)
cd = Pd @ (w * F)
cg = Pg @ (w * F)
lap = np.arange(R + 1) * (np.arange(R + 1) + 1.0)
scale = np.max(np.abs(cl * lap).astype(np.float64))
for name, c in (("reference recurrence (double)", cd), ("GPU scaled recurrence", cg)):
    e = np.abs((c - cl).astype(np.float64)) * lap / scale
    print(f"T{R} r=0 {name}: max |err| * s(s+1) / max|lap c| = {e.max():.2e}; by s-band",
          [f"{e[x:x + (R + 1) // 8].max():.1e}" for x in range(0, R + 1, (R + 1) // 8)])
e = np.abs(cd - cg) * lap / scale
print(f"T{R} r=0 GPU vs reference: {e.max():.2e}")
