import torch, time
dev = torch.device('cuda')
n = 15 * 256 * 256
for trial in range(3):
    h = torch.empty(n, dtype=torch.complex128).pin_memory()
    d = torch.empty(n, dtype=torch.complex128, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    e0.record()
    for _ in range(20): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / 20
    print(f"trial {trial}: H2D {16*n/ms/1e6:.1f} GB/s  D2H {16*n/ms2/1e6:.1f} GB/s")
