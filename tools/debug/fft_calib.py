import torch, time
dev = torch.device('cuda')
for (n, batch) in ((768, 2880), (512, 128 * 64 * 7), (192, 48 * 7)):
    x = torch.randn(batch, n, dtype=torch.complex128, device=dev)
    for _ in range(3): y = torch.fft.fft(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): y = torch.fft.fft(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 5 * n * __import__('math').log2(n) * batch
    print(f"cuFFT Z2Z n={n} batch={batch}: {ms*1e3:.1f} us, {flops/ms/1e9:.2f} TFLOP/s, {2*16*n*batch/ms/1e6:.0f} GB/s")
