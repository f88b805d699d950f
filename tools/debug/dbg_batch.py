import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
from paper_1805_07923_b200 import mlsdc, sdc, swe, workloads
params = swe.ModelParams(**workloads.EARTH)
def rel(a, b): return float(np.max(np.abs(a-b))/np.max(np.abs(b)))
x = np.stack([workloads.seeded_state(31, k) for k in range(3)])
hier = mlsdc.build_hierarchy(params, 31, 5, 15, 3, grid_fine=(96, 48), grid_coarse=(48, 24))
xb = swe.PrognosticState(torch.as_tensor(x).cuda())
for lvl, xx in ((hier.fine, xb), (hier.coarse, xb.truncated(15))):
    for trial in range(3):
        fb = lvl.rhs.eval_f_e(xx).numpy()
        fs = [lvl.rhs.eval_f_e(swe.PrognosticState(xx.data[m].clone())).numpy() for m in range(3)]
        print('fe', lvl.truncation, trial, [rel(fb[m], fs[m]) for m in range(3)])
# sweep
def sweep_test(lvl, xx):
    swb = sdc.initialize_nodes(xx, lvl.rhs, lvl.n_nodes)
    sdc.sdc_sweep(swb, lvl.tables, 240.0, lvl.rhs)
    out = []
    for m in range(3):
        sw1 = sdc.initialize_nodes(swe.PrognosticState(xx.data[m].clone()), lvl.rhs, lvl.n_nodes)
        sdc.sdc_sweep(sw1, lvl.tables, 240.0, lvl.rhs)
        out.append(rel(swb.theta[-1].numpy()[m], sw1.theta[-1].numpy()))
    return out
print('sweep fine', sweep_test(hier.fine, xb))
print('sweep coarse', sweep_test(hier.coarse, xb.truncated(15)))
