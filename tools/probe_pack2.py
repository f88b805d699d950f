import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_07923_b200 import spharm, workloads
R, NF = 255, 15
c_host = torch.from_numpy(workloads.transform_batch(R, NF)).pin_memory()
c_dev = c_host.cuda()
for _ in range(3):
    spharm.upload_coeffs(c_host, out=c_dev)
torch.cuda.synchronize()
print("---- timed", file=sys.stderr, flush=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
a.record()
for _ in range(8):
    spharm.upload_coeffs(c_host, out=c_dev)
b.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print("issue us/upload", (t1 - t) / 8 * 1e6, "gpu us/upload", a.elapsed_time(b) / 8 * 1e3)
