import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_1805_07923_b200 import _lib
lib = _lib.load()
R, nm = 255, 15
T1 = (R + 1) * (R + 2) // 2
src_p = torch.randn(nm, R + 1, R + 1, 2, dtype=torch.float64)
dst_p = torch.empty(nm, T1, 2, dtype=torch.float64)
src_pin, dst_pin = src_p.pin_memory(), dst_p.pin_memory()
torch.zeros(1).cuda()
def t(name, s, d, n=50):
    for _ in range(5):
        lib.swsdc_pack_triangles(s.data_ptr(), R, nm, d.data_ptr())
    t0 = time.perf_counter()
    for _ in range(n):
        lib.swsdc_pack_triangles(s.data_ptr(), R, nm, d.data_ptr())
    print(name, round((time.perf_counter() - t0) / n * 1e6, 1), "us", flush=True)
for rep in range(2):
    t("pageable->pageable", src_p, dst_p)
    t("pinned->pageable", src_pin, dst_p)
    t("pageable->pinned", src_p, dst_pin)
    t("pinned->pinned", src_pin, dst_pin)
a = np.empty(T1 * nm * 2); b = np.empty_like(a)
t0 = time.perf_counter()
for _ in range(50): np.copyto(b, a)
print("np.copyto 7.9MB 1 thread", round((time.perf_counter() - t0) / 50 * 1e6, 1), "us")
print(open('/proc/cpuinfo').read().count('processor'), os.sched_getaffinity(0))
try: print(open('/sys/fs/cgroup/cpu.max').read())
except Exception as e: print(e)
