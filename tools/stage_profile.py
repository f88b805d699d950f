"""Per-stage device time of one MLSDC step (eager, in-library CUDA events)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1805_07923_b200 import _lib, mlsdc, swe, workloads

for name in sys.argv[1:] or ["config0", "config2", "config4"]:
    Rf, gf, Rc, gc, nf, nc, n_it, ncs, dt, steps, members = bench.MLSDC_CONFIGS[name]
    params = swe.ModelParams(**workloads.EARTH)
    hier = mlsdc.build_hierarchy(params, Rf, nf, Rc, nc, grid_fine=gf, grid_coarse=gc)
    x = np.stack([workloads.seeded_state(Rf, k) for k in range(members)]) if members > 1 \
        else workloads.seeded_state(Rf, 0)
    st = swe.PrognosticState(torch.as_tensor(x).cuda())
    mlsdc.mlsdc_timestep(st, dt, n_it, hier, ncs)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mlsdc.mlsdc_timestep(st, dt, n_it, hier, ncs)
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    tot = sum(v[1] for v in prof.values())
    print(f"== {name}: eager step {e0.elapsed_time(e1):.3f} ms, kernel sum {tot:.3f} ms, launches {sum(v[0] for v in prof.values())}")
    for k, (n, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:26s} {n:5d} launches {ms:9.3f} ms  {1e3 * ms / n:8.1f} us/launch")
