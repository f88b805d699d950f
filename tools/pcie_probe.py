"""PCIe probe for the config-1 e2e path: copy-engine and zero-copy bandwidth,
alone and concurrent, for one 15-field T255 batch (7.9 MB triangle, 15.8 MB dense)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_07923_b200 import spharm, workloads

R, NF = 255, 15
c_host = torch.from_numpy(workloads.transform_batch(R, NF)).pin_memory()
o_host = torch.zeros_like(c_host).pin_memory()
c_dev = c_host.cuda()
o_dev = torch.empty_like(c_dev)
dense = c_host.numel() * 16
tri = NF * (R + 1) * (R + 2) // 2 * 16
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}

def timed(name, fns, nbytes, reps=20):
    for _ in range(3):
        for s, f in fns:
            with torch.cuda.stream(s):
                f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    a.record(main)
    for s, _ in fns:
        s.wait_stream(main)
    for _ in range(reps):
        for s, f in fns:
            with torch.cuda.stream(s):
                f()
    for s, _ in fns:
        main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    res[name] = {"us": round(us, 1), "GBps_per_stream": round(nbytes / us / 1e3, 1)}
    print(name, res[name], flush=True)

h2d_dense = lambda: c_dev.copy_(c_host, non_blocking=True)
d2h_dense = lambda: o_host.copy_(o_dev, non_blocking=True)
up_tri = lambda: spharm.upload_coeffs(c_host, out=c_dev)
dn_tri = lambda: spharm.download_coeffs(o_dev, o_host, write_lower=False)
half = c_host.numel() // 2
h2d_half = lambda: c_dev.view(-1)[:half].copy_(c_host.view(-1)[:half], non_blocking=True)
d2h_half = lambda: o_host.view(-1)[:half].copy_(o_dev.view(-1)[:half], non_blocking=True)
timed("h2d dense CE", [(s1, h2d_dense)], dense)
timed("d2h dense CE", [(s1, d2h_dense)], dense)
timed("h2d+d2h dense CE concurrent", [(s1, h2d_dense), (s2, d2h_dense)], dense)
timed("h2d half-size contiguous CE", [(s1, h2d_half)], tri)
timed("d2h half-size contiguous CE", [(s1, d2h_half)], tri)
timed("h2d+d2h half contiguous concurrent", [(s1, h2d_half), (s2, d2h_half)], tri)
timed("upload triangle zero-copy", [(s1, up_tri)], tri)
timed("download triangle staircase", [(s1, dn_tri)], tri)
timed("upload tri + download tri concurrent", [(s1, up_tri), (s2, dn_tri)], tri)
timed("upload tri + d2h half concurrent", [(s1, up_tri), (s2, d2h_half)], tri)
timed("h2d half contiguous + download tri concurrent", [(s1, h2d_half), (s2, dn_tri)], tri)
timed("h2d half contiguous + download tri + upload tri", [(s1, h2d_half), (s2, dn_tri)], tri)
json.dump(res, open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "pcie_probe_%s.json" % os.environ.get("PROBE_TAG", "default")), "w"), indent=1)
