"""Phase timeline of the fused F_E grid kernel (swe_grid_reg_kernel) from a
trace build of fourier.cu (nvcc ... -DGRID_TRACE, linked as abtest/lib_gtrace.so,
used via SWSDC_LIB): per-CTA %globaltimer stamps 0 entry, 1 rings filled,
2 inverse FFTs done, 3 products done, 4 forward FFTs done, 5 cluster barrier
passed, 6 outputs written, 7 exit barrier passed.  Usage: grid_trace.py R n_lon
n_lat members."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1805_07923_b200 import _lib, spharm, swe, workloads

R, I, J, M = (int(v) for v in sys.argv[1:5])
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
rhs = swe.ShallowWaterRHS(plan, swe.ModelParams(**workloads.EARTH))
x = np.stack([workloads.seeded_state(R, k) for k in range(M)]) if M > 1 else workloads.seeded_state(R, 0)
st = swe.PrognosticState(torch.as_tensor(x).cuda())
fn = _lib.load().swsdc_debug_grid_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(3):
    rhs.eval_f_e(st)
torch.cuda.synchronize()
fn(None, 1)
torch.cuda.synchronize()
rhs.eval_f_e(st)
torch.cuda.synchronize()
buf = np.zeros((16384, 8), dtype=np.uint64)
fn(buf.ctypes.data, 0)
t = buf.astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
t = np.where(t > 0, t - t0, -1)
names = ["entry", "filled", "inverse", "products", "forward", "cluster", "output", "exit"]
print(f"R={R} grid {I}x{J} members {M}: CTAs {len(t)}, span {t.max()} ns")
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (4, 6), (0, 6), (0, 7), (1, 5), (5, 7), (7, 2)]:
    m = (t[:, a] >= 0) & (t[:, b] >= 0)
    d = t[m, b] - t[m, a]
    if d.size == 0:
        continue
    print(f"  {names[a]:>8s} -> {names[b]:8s}: med {int(np.median(d)):7d} ns  p10 {int(np.percentile(d, 10)):7d}  p90 {int(np.percentile(d, 90)):7d}")
