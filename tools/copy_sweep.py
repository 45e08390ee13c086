"""HBM copy bandwidth vs buffer size (torch copy_, back-to-back, CUDA events): the
practical ceiling for a per-GPU stencil share of that size.  Not part of the library."""
import torch

torch.cuda.init()
for mb in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096):
    n = mb * (1 << 20) // 8
    a = torch.empty(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    for _ in range(5):
        b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 200
    e0.record()
    for _ in range(it):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / it
    print(f"{mb:5d} MiB per buffer: {us:8.1f} us/copy  {2 * mb * (1 << 20) / us / 1e3:7.0f} GB/s")
