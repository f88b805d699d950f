import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import swsdc_oracle as orc
from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads
params = swe.ModelParams(**workloads.EARTH); op = orc.OracleParams(**workloads.EARTH)
def rel(a, b): return np.max(np.abs(a-b))/np.max(np.abs(b))
oh = orc.OracleHierarchy(orc.OracleLevel(31, 5, op, (96, 48)), orc.OracleLevel(15, 3, op, (48, 24)))
x = np.stack([workloads.seeded_state(31, k) for k in range(3)])
want = [orc.mlsdc_step(x[m], 240.0, 2, oh, coarse_sweeps=2) for m in range(3)]
for members in (1, 3):
    for graph in (False, True):
        hier = mlsdc.build_hierarchy(params, 31, 5, 15, 3, grid_fine=(96, 48), grid_coarse=(48, 24))
        xs = x[:members] if members > 1 else x[0]
        st = stepper.MLSDCStepper(hier, 240.0, 2, swe.PrognosticState(torch.as_tensor(xs).cuda()), n_coarse_sweeps=2, use_graph=graph)
        y = st.run(1).numpy()
        if members == 1: y = y[None]
        print(members, graph, [rel(y[m], want[m]) for m in range(members)])
# direct eager batched mlsdc_timestep
hier = mlsdc.build_hierarchy(params, 31, 5, 15, 3, grid_fine=(96, 48), grid_coarse=(48, 24))
y = mlsdc.mlsdc_timestep(swe.PrognosticState(torch.as_tensor(x).cuda()), 240.0, 2, hier, 2).numpy()
print('eager batched', [rel(y[m], want[m]) for m in range(3)])
# batched eval_fe vs per member
rhs = hier.fine.rhs
xb = swe.PrognosticState(torch.as_tensor(x).cuda())
fb = rhs.eval_f_e(xb).numpy()
orhs = orc.OracleRHS(orc.OraclePlan(31, 96, 48), op)
print('fe batched', [rel(fb[m], orhs.eval_fe(x[m])) for m in range(3)])
fi = rhs.eval_f_i(xb).numpy()
print('fi batched', [rel(fi[m], orhs.eval_fi(x[m])) for m in range(3)])
so = rhs.solve_implicit(xb, 100.0).numpy()
print('solve batched', [rel(so[m], orhs.solve(x[m], 100.0)) for m in range(3)])
tr = xb.truncated(15).numpy()
print('trunc', [rel(tr[m], orc.trunc(x[m], 15)) for m in range(3)])
