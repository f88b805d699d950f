"""CPU issue cost of the e2e step vs its GPU time (config 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm

R, I, J, NF, NG = 255, 768, 384, 15, 3
gsz = NF // NG
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
plan.reserve(gsz)
c = torch.randn(NF, R + 1, R + 1, dtype=torch.complex128).triu()
c_pin = c.pin_memory(); o_pin = torch.empty_like(c_pin).pin_memory()
c_dev = c.cuda(); g = plan.synthesize(c_dev); out = plan.analyze(g)
s_in, s_cmp, s_out = (torch.cuda.Stream() for _ in range(3))
def step():
    main = torch.cuda.current_stream()
    ev_in = [torch.cuda.Event() for _ in range(NG)]
    ev_cmp = [torch.cuda.Event() for _ in range(NG)]
    s_in.wait_stream(main); s_cmp.wait_stream(main); s_out.wait_stream(main)
    for gi in range(NG):
        sl = slice(gi * gsz, (gi + 1) * gsz)
        with torch.cuda.stream(s_in):
            spharm.upload_coeffs(c_pin[sl], out=c_dev[sl]); ev_in[gi].record(s_in)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in[gi])
            plan.synthesize(c_dev[sl], out=g[sl]); plan.analyze(g[sl], out=out[sl])
            ev_cmp[gi].record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[gi]); o_pin[sl].copy_(out[sl], non_blocking=True)
    main.wait_stream(s_out)
for _ in range(5): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"issue {1e3*(t1-t0)/50:.3f} ms/step, wall {1e3*(t2-t0)/50:.3f} ms/step")
t0 = time.perf_counter()
for _ in range(200): plan.synthesize(c_dev[:5], out=g[:5])
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"synthesize call {1e6*(t1-t0)/200:.1f} us")
t0 = time.perf_counter()
for _ in range(200): spharm.upload_coeffs(c_pin[:5], out=c_dev[:5])
t1 = time.perf_counter()
print(f"upload call {1e6*(t1-t0)/200:.1f} us")
torch.cuda.synchronize()
# graph-captured step
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    step()
gr.replay(); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(50): gr.replay()
e.record(); torch.cuda.synchronize()
print(f"graph replay {s.elapsed_time(e)/50:.3f} ms/step")
