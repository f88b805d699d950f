"""Where does the GPU F_E deviate from the streaming oracle at large R?"""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1805_07923_b200 import spharm, swe, workloads
import swsdc_oracle as orc, swsdc_stream as stm

ROWS = np.array([0, 1, 31, 32, 33, 127, 255, 511, 640, 1023, 1151, 1278, 1279])
g = np.load(os.path.join(ROOT, "tests/golden/large_t1279.npz"))
plan = spharm.TransformPlan(spharm.build_gaussian_grid(1920, 3840), 1279)
rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**workloads.EARTH))
x = workloads.seeded_state(1279, 0)
fe = rhs.eval_f_e(swe.PrognosticState(x)).numpy()
for f in range(3):
    sc = g["fe_seed0_absmax"][f]
    d = np.abs(fe[f][ROWS] - g["fe_seed0_rows"][f]) / sc
    print("field", f, "absmax", sc)
    for i, r in enumerate(ROWS):
        s = np.argmax(d[i]); print(f"  r={r}: max rel {d[i].max():.2e} at s={s}; |want| there {abs(g['fe_seed0_rows'][f][i][s])/sc:.2e}; err over s-bands",
              [f"{d[i][a:a+160].max():.1e}" for a in range(0, 1280, 160)])
# T639 live comparison, linear and nonlinear
for R, I, J in ((639, 1920, 960),):
    p2 = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
    sp = stm.StreamPlan(R, I, J)
    x = workloads.seeded_state(R, 0)
    for nl in (False, True):
        r2 = swe.ShallowWaterRHS(p2, swe.ModelParams(**workloads.EARTH), include_nonlinear=nl)
        got = r2.eval_f_e(swe.PrognosticState(x)).numpy()
        t = time.time()
        want = stm.StreamRHS(sp, orc.OracleParams(**workloads.EARTH), nl).eval_fe(x)
        for f in range(3):
            if np.max(np.abs(want[f])) == 0: continue
            d = np.abs(got[f] - want[f]) / np.max(np.abs(want[f]))
            r, s = np.unravel_index(np.argmax(d), d.shape)
            print(f"T{R} nl={nl} field {f}: {d.max():.2e} at r={r} s={s} (oracle {time.time()-t:.0f}s)")
    # separate pieces: eval_n composed path
    r2 = swe.ShallowWaterRHS(p2, swe.ModelParams(**workloads.EARTH))
    n = r2.eval_n(swe.PrognosticState(x)).numpy()
    orhs = stm.StreamRHS(sp, orc.OracleParams(**workloads.EARTH), True)
    lin = stm.StreamRHS(sp, orc.OracleParams(**workloads.EARTH), False)
    wn = orhs.eval_fe(x) - lin.eval_fe(x)
    for f in range(3):
        d = np.abs(n[f] - wn[f]) / np.max(np.abs(wn[f]))
        r, s = np.unravel_index(np.argmax(d), d.shape)
        print(f"T{R} eval_n field {f}: {d.max():.2e} at r={r} s={s}")
