"""Copy-engine peer copy (GPU1 -> GPU0, 256 MiB, the 2MM ROW D block at N=2) timed
alone and while both GPUs run bf16 GEMMs (torch.matmul) on other streams: does a
GPU-filling product slow the NVLink copy down?"""
import torch

n = 16384
src = torch.empty(8192 * n, dtype=torch.bfloat16, device="cuda:1").fill_(1)
dst = torch.empty(8192 * n, dtype=torch.bfloat16, device="cuda:0")
a = [torch.randn(8192, n, device=f"cuda:{d}", dtype=torch.bfloat16) for d in (0, 1)]
b = [torch.randn(n, n, device=f"cuda:{d}", dtype=torch.bfloat16) for d in (0, 1)]
cs = torch.cuda.Stream(device="cuda:0")
gs = [torch.cuda.Stream(device=f"cuda:{d}") for d in (0, 1)]


def copy_ms(busy):
    for d in (0, 1):
        torch.cuda.synchronize(d)
    if busy:
        for d in (0, 1):
            with torch.cuda.device(d), torch.cuda.stream(gs[d]):
                for _ in range(3):
                    torch.matmul(a[d], b[d])
    with torch.cuda.device(0), torch.cuda.stream(cs):
        torch.cuda._sleep(2_000_000)  # ~1 ms: let the GEMMs get going
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        dst.copy_(src, non_blocking=True)
        e1.record(cs)
    for d in (0, 1):
        torch.cuda.synchronize(d)
    return e0.elapsed_time(e1)


for busy in (False, True, False, True):
    ts = sorted(copy_ms(busy) for _ in range(5))
    ms = ts[2]
    print(f"busy={busy}: copy {ms:.3f} ms = {src.numel() * 2 / ms / 1e6:.0f} GB/s (median of 5)")


def gemm_ms(with_copy):
    """3 GEMMs on GPU0 alone, or with the 256 MiB peer copy (and GPU1's GEMMs) alongside."""
    for d in (0, 1):
        torch.cuda.synchronize(d)
    with torch.cuda.device(0), torch.cuda.stream(gs[0]):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs[0])
        for _ in range(3):
            torch.matmul(a[0], b[0])
        e1.record(gs[0])
    if with_copy:
        with torch.cuda.device(1), torch.cuda.stream(gs[1]):
            for _ in range(3):
                torch.matmul(a[1], b[1])
        with torch.cuda.device(0), torch.cuda.stream(cs):
            for _ in range(3):  # ~1.1 ms of copies over the ~7.5 ms of products
                dst.copy_(src, non_blocking=True)
    for d in (0, 1):
        torch.cuda.synchronize(d)
    return e0.elapsed_time(e1)


for wc in (False, True, False, True):
    ts = sorted(gemm_ms(wc) for _ in range(5))
    print(f"with_copy={wc}: 3 GEMMs {ts[2]:.3f} ms (median of 5)")
