"""One CUDA-graph MLSDC step of a bench config inside an NVTX range "step" (for ncu --nvtx)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1805_07923_b200 import mlsdc, stepper, swe, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
Rf, gf, Rc, gc, nf, nc, n_it, ncs, dt, steps, members = bench.MLSDC_CONFIGS[name]
params = swe.ModelParams(**workloads.EARTH)
hier = mlsdc.build_hierarchy(params, Rf, nf, Rc, nc, grid_fine=gf, grid_coarse=gc)
x = np.stack([workloads.seeded_state(Rf, k) for k in range(members)]) if members > 1 \
    else workloads.seeded_state(Rf, 0)
st = swe.PrognosticState(torch.as_tensor(x).cuda())
stp = stepper.MLSDCStepper(hier, dt, n_it, st, n_coarse_sweeps=ncs)
stp.run(3)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); stp.run(10); e.record(); torch.cuda.synchronize()
print(f"{name}: graph step {s.elapsed_time(e) / 10:.3f} ms")
torch.cuda.nvtx.range_push("step")
stp.run(1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
