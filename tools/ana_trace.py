"""Phase timeline of the DMMA analysis kernel at config 1 from a trace build of
legendre.cu (nvcc ... -DANA_TRACE, linked as abtest/lib_trace.so, used via SWSDC_LIB):
stamps 0 entry, 1 tables loaded, 2 first q tile done, 3 first x fragments
arrived, 4 k-loop done, 5 reduction done, 6 epilogue stored."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1805_07923_b200 import _lib, spharm, workloads

R, I, J, NF = 255, 768, 384, 15
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
c = torch.as_tensor(workloads.transform_batch(R, NF)).cuda()
g = plan.synthesize(c)
out = plan.analyze(g)
lib = _lib.load()
fn = lib.swsdc_debug_ana_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(3):
    plan.analyze(g, out=out)
torch.cuda.synchronize()
fn(None, 1)
torch.cuda.synchronize()
plan.analyze(g, out=out)
torch.cuda.synchronize()
buf = np.zeros((16384, 8), dtype=np.uint64)
fn(buf.ctypes.data, 0)
t = buf[:, :7].astype(np.int64)
valid = t[:, 0] > 0
t = t[valid]
t0 = t[:, 0].min()
t = np.where(t > 0, t - t0, -1)
print("warps traced", len(t), "kernel span (ns)", t[:, 6].max() if (t[:, 6] >= 0).any() else None)
names = ["entry", "tables", "q tile", "first x", "k-loop end", "reduction", "stored"]
for k in range(7):
    col = t[:, k][t[:, k] >= 0]
    if len(col):
        print(f"  stamp {k} {names[k]:11s} n={len(col):5d} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d}")
act = (t[:, 1] >= 0) & (t[:, 4] >= 0)
d = t[act]
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (0, 6)]:
    m = (d[:, a] >= 0) & (d[:, b] >= 0)
    x = d[m, b] - d[m, a]
    if len(x):
        print(f"  {names[a]:>10s} -> {names[b]:11s}: med {int(np.median(x)):6d} ns  p90 {int(np.percentile(x, 90)):6d}  max {x.max():6d}")
# start-time histogram: how many warps start in each 2 us bin
st = d[:, 0]
h, e = np.histogram(st, bins=np.arange(0, st.max() + 2000, 2000))
print("  warp start histogram (2 us bins):", h.tolist())
