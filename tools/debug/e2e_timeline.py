"""Per-piece start/end (us, relative to step start) of the e2e pipeline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm

R, I, J, NF = 255, 768, 384, 15
NG = int(sys.argv[1]) if len(sys.argv) > 1 else 3
gsz = NF // NG
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
plan.reserve(gsz)
c = torch.randn(NF, R + 1, R + 1, dtype=torch.complex128).triu()
c_pin = c.pin_memory(); o_pin = torch.empty_like(c_pin).pin_memory()
c_dev = c.cuda(); g = plan.synthesize(c_dev); out = plan.analyze(g)
s_in, s_cmp, s_out = (torch.cuda.Stream() for _ in range(3))
E = lambda: torch.cuda.Event(enable_timing=True)
def step(marks):
    main = torch.cuda.current_stream()
    t0 = E(); t0.record(main); marks.append(("t0", t0))
    s_in.wait_stream(main); s_cmp.wait_stream(main); s_out.wait_stream(main)
    up_done = []
    with torch.cuda.stream(s_in):
        for gi in range(NG):
            sl = slice(gi * gsz, (gi + 1) * gsz)
            a, b = E(), E()
            a.record(s_in); spharm.upload_coeffs(c_pin[sl], out=c_dev[sl]); b.record(s_in)
            marks.append((f"U{gi}", a, b)); up_done.append(b)
    for gi in range(NG):
        sl = slice(gi * gsz, (gi + 1) * gsz)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(up_done[gi])
            a, m, b = E(), E(), E()
            a.record(s_cmp); plan.synthesize(c_dev[sl], out=g[sl]); m.record(s_cmp)
            plan.analyze(g[sl], out=out[sl]); b.record(s_cmp)
            marks.append((f"S{gi}", a, m)); marks.append((f"A{gi}", m, b))
        with torch.cuda.stream(s_out):
            s_out.wait_event(b)
            a2, b2 = E(), E()
            a2.record(s_out); spharm.download_coeffs(out[sl], o_pin[sl], write_lower=False); b2.record(s_out)
            marks.append((f"D{gi}", a2, b2))
    main.wait_stream(s_out)
for _ in range(3):
    step([])
torch.cuda.synchronize()
marks = []
step(marks)
torch.cuda.synchronize()
t0 = marks[0][1]
for name, a, b in marks[1:]:
    print(f"{name:4s} {1e3 * t0.elapsed_time(a):7.1f} {1e3 * t0.elapsed_time(b):7.1f}")
