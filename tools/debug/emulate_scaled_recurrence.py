"""CPU experiment: does the GPU's scaled recurrence (q_s = mu q_{s-1} - beta_s q_{s-2},
P_s = g_s q_s, restarted from exact checkpoint seeds every 32 degrees) explain the
r = 0 deviation of the GPU F_E from the reference at large R?  Emulates the GPU
tables in numpy (fma via long double) and compares F_E against the exact-table
streaming oracle."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import swsdc_oracle as orc, swsdc_stream as stm
from paper_1805_07923_b200 import workloads

K = 32
EXACT_ROWS = int(os.environ.get("EXACT_ROWS", "0"))


class EmuPlan(stm.StreamPlan):
    def _p_block(self, r0, r1):
        P = super()._p_block(r0, r1)          # exact reference tables (seeds)
        mu = self.mu.astype(np.longdouble)
        out = P.copy()
        for i in range(r1 - r0):
            r = r0 + i
            if r < EXACT_ROWS:
                continue
            smax = self.R + 1
            s = np.arange(r, smax + 1)
            a = np.zeros(s.size); b = np.zeros(s.size)
            a[1] = np.sqrt(2.0 * r + 3.0)
            ss = s[2:]
            s2r2 = (ss * ss - r * r).astype(float)
            a[2:] = np.sqrt((4.0 * ss * ss - 1.0) / s2r2)
            b[2:] = np.sqrt((2.0 * ss + 1.0) * (ss - 1.0 - r) * (ss - 1.0 + r) / ((2.0 * ss - 3.0) * s2r2))
            beta = np.zeros(s.size); beta[2:] = b[2:] / (a[2:] * a[1:-1])
            g = np.ones(s.size)
            for k in range(1, s.size):
                g[k] = 1.0 if k % K == 0 else g[k - 1] * a[k]
            n = s.size
            for k0 in range(0, n, K):
                qa = P[i, r - r0 + k0]                       # seed P_{k0}
                if k0 + 1 >= n:
                    break
                qb = P[i, r - r0 + k0 + 1] / a[k0 + 1]       # seed P_{k0+1}/a_{k0+1}
                out[i, r - r0 + k0 + 1] = qb * g[k0 + 1]
                for k in range(k0 + 2, min(k0 + K, n)):
                    t = (-beta[k]) * qa
                    qn = (mu * qb.astype(np.longdouble) + t).astype(np.float64)
                    out[i, r - r0 + k] = qn * g[k]
                    qa, qb = qb, qn
        return out


R, I, J = int(sys.argv[1]) if len(sys.argv) > 1 else 639, 0, 0
I, J = {255: (768, 384), 639: (1920, 960), 1279: (3840, 1920)}[R]
x = workloads.seeded_state(R, 0)
prm = orc.OracleParams(**workloads.EARTH)
t = time.time()
want = stm.StreamRHS(stm.StreamPlan(R, I, J), prm).eval_fe(x)
got = stm.StreamRHS(EmuPlan(R, I, J), prm).eval_fe(x)
print(f"{time.time()-t:.0f}s EXACT_ROWS={EXACT_ROWS}")
for f in range(3):
    d = np.abs(got[f] - want[f]) / np.max(np.abs(want[f]))
    r, s = np.unravel_index(np.argmax(d), d.shape)
    print(f"field {f}: {d.max():.2e} at r={r} s={s}; rows 0..4 max:", [f"{d[k].max():.1e}" for k in range(5)], "r>=5:", f"{d[5:].max():.1e}")
