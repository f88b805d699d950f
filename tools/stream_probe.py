"""Probe: config-1 transform pair (15 T255 fields) on one stream vs the batch
split over 2-3 concurrent streams (one plan per stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_07923_b200 import spharm, workloads

R, I, J = 255, 768, 384
grid = spharm.build_gaussian_grid(J, I)
plans = [spharm.TransformPlan(grid, R) for _ in range(3)]
c = torch.as_tensor(workloads.transform_batch(R, 15)).cuda()
streams = [torch.cuda.Stream() for _ in range(3)]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

def run(splits):
    main = torch.cuda.current_stream()
    ev0 = torch.cuda.Event()
    ev0.record(main)
    ends = []
    lo = 0
    for k, n in enumerate(splits):
        s = streams[k]
        s.wait_event(ev0)
        with torch.cuda.stream(s):
            g = plans[k].synthesize(c[lo:lo + n])
            plans[k].analyze(g)
            e = torch.cuda.Event()
            e.record(s)
            ends.append(e)
        lo += n
    for e in ends:
        main.wait_event(e)

for splits in ([15], [10, 5], [5, 5, 5], [8, 7], [15], [10, 5], [5, 5, 5], [8, 7]):
    for _ in range(3):
        run(splits)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); run(splits); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(splits, f"median {ts[len(ts)//2]*1e3:.1f} us  min {ts[0]*1e3:.1f} us")
