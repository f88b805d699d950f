"""Validate the streaming oracle against the REFERENCE, then use it for T1279.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_large.py [validate] [t1279] [step]

* validate -- oracle/swsdc_stream.py against the reference's own dense
  TransformPlan / ShallowWaterRHS (spharm.py, swe.py) at T255 on 384x768 and
  T639 on 960x1920 (the largest plan the reference can build here: 14.4 GB):
  synthesize, analyze, the vector transforms and F_E.  The relative L-inf
  deviations are stored in `large_validation.npz`: <= 1e-14 for the
  transforms, <= 1e-13 for F_E (its delta tendency cancels large terms, so
  the blocked matmuls' different summation order shows at ~4e-14 of the
  field maximum at T639), and exactly 0 for F_E with one block spanning all
  r (same matmuls as the reference: every table entry is bitwise equal).
* t1279 -- BASELINE configs[3] fine grid, T1279 on 1920x3840, from the
  validated streaming oracle (the reference's dense tables would need
  126 GB): synthesize of the seed-0 phi' field (longitude columns), the
  synthesize->analyze pair, analyze of a seeded noise grid, and F_E of the
  seed-0 state.
* step -- one config-3 MLSDC(3,2,2) step T1279/T639, dt=60, seed 0.

Spectral outputs at T1279 are too large to commit whole (13 MB per field), so
each is stored as (i) the full rows at ROWS (every 32-degree checkpoint
neighbourhood the GPU recurrence restarts from is represented, plus both ends)
and (ii) for EVERY row r, four seeded projections sum_s c[r, s] v_k[s]
(`proj`), which any wrong coefficient perturbs.  Tests rebuild v_k from the
seed.  Outputs: `large_t1279.npz`, `large_step.npz`.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, HERE)

import swsdc_oracle as orc  # noqa: E402
import swsdc_stream as stm  # noqa: E402

from paper_1805_07923_b200 import workloads  # noqa: E402

ROWS = np.array([0, 1, 31, 32, 33, 127, 255, 511, 640, 1023, 1151, 1278, 1279])
PROJ_SEED = 777


def proj_vectors(R: int) -> np.ndarray:
    return np.random.default_rng(PROJ_SEED).normal(size=(4, R + 1))


def compact(prefix: str, c: np.ndarray, out: dict) -> None:
    """Rows at ROWS plus per-row projections of a (..., R+1, R+1) array."""
    R = c.shape[-1] - 1
    out[f"{prefix}_rows"] = c[..., ROWS, :]
    out[f"{prefix}_proj"] = c @ proj_vectors(R).T
    out[f"{prefix}_absmax"] = np.max(np.abs(c), axis=(-2, -1))


def cols(I: int) -> np.ndarray:
    return np.array([0, 1, I // 7, I // 3 + 1, I // 2, I - 1])


def noise_grid(seed: int, I: int, J: int) -> np.ndarray:
    return np.random.default_rng(seed).normal(size=(I, J))


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def validate():
    sys.path.insert(0, "/root/reference/pkg/src")
    from swsdc import spharm  # reference, read-only
    from swsdc.swe import ModelParams, PrognosticState, ShallowWaterRHS
    out = {}
    for R, I, J in ((255, 768, 384), (639, 1920, 960)):
        t0 = time.time()
        ref = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
        sp = stm.StreamPlan(R, I, J)
        rng = np.random.default_rng(5000 + R)
        c, c2 = (workloads.spectral_noise(rng, R, 1.0, False) for _ in range(2))
        g, g2 = noise_grid(5001 + R, I, J), noise_grid(5002 + R, I, J)
        dev = [rel(sp.synthesize(c), ref.synthesize(c)), rel(sp.analyze(g), ref.analyze(g))]
        dev += [rel(a, b) for a, b in zip(sp.synth_uv(c, c2), ref.synthesize_pair_cos_gradient(c, c2))]
        dev += [rel(a, b) for a, b in zip(sp.anal_divcurl(g, g2), ref.analyze_vector_div_curl(g, g2))]
        x = workloads.seeded_state(R, 0)
        rr = ShallowWaterRHS(ref, ModelParams(**workloads.EARTH))
        fe_ref = rr.eval_f_e(PrognosticState(x[0].copy(), x[1].copy(), x[2].copy()))
        fe = stm.StreamRHS(sp, orc.OracleParams(**workloads.EARTH)).eval_fe(x)
        dev += [rel(fe[0], fe_ref.phi_prime), rel(fe[1], fe_ref.zeta), rel(fe[2], fe_ref.delta)]
        # one block spanning every r repeats the reference's matmuls exactly
        sp1 = stm.StreamPlan(R, I, J, block_bytes=1e12)
        fe1 = stm.StreamRHS(sp1, orc.OracleParams(**workloads.EARTH)).eval_fe(x)
        dev += [float(np.max(np.abs(fe1 - np.stack([fe_ref.phi_prime, fe_ref.zeta, fe_ref.delta]))))]
        out[f"dev_R{R}"] = np.array(dev)
        print(f"R={R}: deviations ({time.time() - t0:.1f} s)", dev)
        assert max(dev[:6]) <= 1e-14, dev      # transforms
        assert max(dev[6:9]) <= 1e-13, dev     # F_E: blocked matmul summation order
        assert dev[9] == 0.0, dev              # bitwise with a single block
        del ref
    np.savez_compressed(os.path.join(HERE, "large_validation.npz"), **out)


def t1279():
    R, I, J = 1279, 3840, 1920
    sp = stm.StreamPlan(R, I, J)
    x = workloads.seeded_state(R, 0)
    out = {}
    t0 = time.time()
    g = sp.synthesize(x[0])
    out["syn_phi_cols"] = g[cols(I)]
    compact("pair_phi", sp.analyze(g), out)
    print(f"pair {time.time() - t0:.1f} s")
    compact("ana_noise", sp.analyze(noise_grid(12791, I, J)), out)
    print(f"noise {time.time() - t0:.1f} s")
    fe = stm.StreamRHS(sp, orc.OracleParams(**workloads.EARTH)).eval_fe(x)
    compact("fe_seed0", fe, out)
    print(f"fe {time.time() - t0:.1f} s")
    np.savez_compressed(os.path.join(HERE, "large_t1279.npz"), **out)


def step():
    prm = orc.OracleParams(**workloads.EARTH)
    h = stm.OracleHierarchy(stm.StreamLevel(1279, 3, prm, (3840, 1920)),
                            stm.StreamLevel(639, 2, prm, (1920, 960)))
    t0 = time.time()
    y = orc.mlsdc_step(workloads.seeded_state(1279, 0), 60.0, 2, h)
    print(f"step {time.time() - t0:.1f} s")
    out = {"counts": np.array([h.fine.rhs.n_solve, h.fine.rhs.n_fi, h.fine.rhs.n_fe,
                               h.coarse.rhs.n_solve, h.coarse.rhs.n_fi, h.coarse.rhs.n_fe])}
    compact("out", y, out)
    np.savez_compressed(os.path.join(HERE, "large_step.npz"), **out)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["validate", "t1279", "step"]
    for p in parts:
        {"validate": validate, "t1279": t1279, "step": step}[p]()
