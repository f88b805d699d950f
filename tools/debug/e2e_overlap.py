"""Which e2e pieces overlap? Pairs of (upload U, compute C, download D) on two streams."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm

R, I, J, NF = 255, 768, 384, 15
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
c = torch.randn(NF, R + 1, R + 1, dtype=torch.complex128).triu()
c_pin = c.pin_memory(); o_pin = torch.empty_like(c_pin).pin_memory()
c_dev = c.cuda(); c2 = c.cuda(); g = plan.synthesize(c_dev); out = plan.analyze(g)
pieces = {
    "U": lambda: spharm.upload_coeffs(c_pin, out=c2),
    "H": lambda: c2.copy_(c_pin, non_blocking=True),
    "C": lambda: (plan.synthesize(c_dev, out=g), plan.analyze(g, out=out)),
    "D": lambda: o_pin.copy_(out, non_blocking=True),
}
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def run(names, reps=20):
    main = torch.cuda.current_stream()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for warm in (True, False):
        torch.cuda.synchronize()
        if not warm: s.record()
        for _ in range(1 if warm else reps):
            sa.wait_stream(main); sb.wait_stream(main)
            for st, n in zip((sa, sb), names):
                with torch.cuda.stream(st):
                    pieces[n]()
            main.wait_stream(sa); main.wait_stream(sb)
        if not warm: e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for n in pieces:
    print(n, f"{run(n):.3f}")
for pair in ("UC", "UD", "CD", "HD", "HC"):
    print(pair, f"{run(pair):.3f}")
