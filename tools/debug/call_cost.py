"""Host cost (us) of the pieces of one TransformPlan.synthesize call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1805_07923_b200 import spharm, _lib

R, I, J = 255, 768, 384
plan = spharm.TransformPlan(spharm.build_gaussian_grid(J, I), R)
c = torch.zeros(5, R + 1, R + 1, dtype=torch.complex128, device="cuda")
g = plan.synthesize(c)
dev = plan.device
lib = _lib.load()
h, st = plan.handle, spharm._stream_ptr(dev)
def t(name, fn, n=5000):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:28s} {1e6 * (time.perf_counter() - t0) / n:7.2f} us")
t("is_pinned_host(dev)", lambda: spharm._is_pinned_host(c))
t("to_device", lambda: spharm._to_device(c, torch.complex128, dev))
t("coeff_in", lambda: plan._coeff_in(c))
t("current_device", torch.cuda.current_device)
t("dev_guard", lambda: spharm._dev_guard(dev))
t("stream_ptr", lambda: spharm._stream_ptr(dev))
t("data_ptr", lambda: c.data_ptr())
t("c[:5] slice", lambda: c[:5])
t("raw lib call (30, idle GPU)", lambda: lib.swsdc_synthesize(h, c.data_ptr(), R, 5, g.data_ptr(), st), 30)
torch.cuda.synchronize()
t("synthesize(out=g) (30)", lambda: plan.synthesize(c, out=g), 30)
torch.cuda.synchronize()
o = plan.analyze(g)
t("analyze(out=o) (30)", lambda: plan.analyze(g, out=o), 30)
torch.cuda.synchronize()
t("upload_coeffs (30)", lambda: spharm.upload_coeffs(c.cpu().pin_memory(), out=c) if False else None, 30)
cp = c.cpu().pin_memory()
t("upload_coeffs (30)", lambda: spharm.upload_coeffs(cp, out=c), 30)
torch.cuda.synchronize()
t("empty kernel torch (30)", lambda: c.zero_(), 30)
torch.cuda.synchronize()
t("event record", lambda: torch.cuda.Event().record())
