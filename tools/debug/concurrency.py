"""Do independent field groups on separate streams overlap the latency-bound kernels?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm

R, I, J, NF = 255, 768, 384, 15
grid = spharm.build_gaussian_grid(J, I)
c = torch.randn(NF, R + 1, R + 1, dtype=torch.complex128, device="cuda").triu()
plans = [spharm.TransformPlan(grid, R) for _ in range(5)]
g = plans[0].synthesize(c); out = plans[0].analyze(g)

def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

def grouped(ng, op):
    gs = NF // ng
    streams = [torch.cuda.Stream() for _ in range(ng)]
    def run():
        main = torch.cuda.current_stream()
        for k, st in enumerate(streams):
            st.wait_stream(main)
            with torch.cuda.stream(st):
                sl = slice(k * gs, (k + 1) * gs)
                if op in ("syn", "pair"): plans[k].synthesize(c[sl], out=g[sl])
                if op in ("ana", "pair"): plans[k].analyze(g[sl], out=out[sl])
        for st in streams: main.wait_stream(st)
    return run

for op in ("syn", "ana", "pair"):
    one = t(grouped(1, op))
    print(f"{op}: 1x15 {one:.1f} us", " ".join(f"{ng}x{NF // ng} {t(grouped(ng, op)):.1f}" for ng in (3, 5)))
