"""Isolated timings of the e2e pieces at config 1 (15 x T255)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm

R, I, J, NF = 255, 768, 384, 15
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
c = torch.randn(NF, R + 1, R + 1, dtype=torch.complex128).triu()
c_pin = c.pin_memory()
o_pin = torch.empty_like(c_pin).pin_memory()
c_dev = c.cuda()
g = plan.synthesize(c_dev)
out = plan.analyze(g)

def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

nb = c.numel() * 16
tri = NF * (R + 1) * (R + 2) // 2 * 16
for ct in (16, 32, 64, 148, 296):
    os.environ["SWSDC_UPLOAD_CTAS"] = str(ct)
print("upload (cap fixed at first call):", end=" ")
ms = t(lambda: spharm.upload_coeffs(c_pin, out=c_dev))
print(f"{ms:.3f} ms  {tri / ms / 1e6:.1f} GB/s triangle")
ms = t(lambda: c_dev.copy_(c_pin, non_blocking=True))
print(f"dense H2D {ms:.3f} ms {nb / ms / 1e6:.1f} GB/s")
ms = t(lambda: o_pin.copy_(out, non_blocking=True))
print(f"dense D2H {ms:.3f} ms {nb / ms / 1e6:.1f} GB/s")
ms = t(lambda: (plan.synthesize(c_dev, out=g), plan.analyze(g, out=out)))
print(f"compute {ms:.3f} ms")
for k in (1, 3, 5):
    sl = slice(0, k)
    ms = t(lambda: c_dev[sl].copy_(c_pin[sl], non_blocking=True))
    print(f"dense H2D {k} fields {ms:.3f} ms {nb * k / NF / ms / 1e6:.1f} GB/s")
    ms = t(lambda: spharm.upload_coeffs(c_pin[sl], out=c_dev[sl]))
    print(f"upload {k} fields {ms:.3f} ms {tri * k / NF / ms / 1e6:.1f} GB/s")
