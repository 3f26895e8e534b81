"""Write-only and copy HBM bandwidth on this GPU (the C2 matrix kernel is write-dominated).

    python tools/hbm_write_bw.py"""
import torch

n = 1536 * 1024 * 1024 // 8  # 1.5 GiB of fp64, like the C2 element matrices
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn, nbytes in (("fill (write only)", lambda: a.fill_(1.0), 8 * n),
                         ("copy (read + write)", lambda: b.copy_(a), 16 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name:22s} {nbytes / best / 1e6:8.1f} GB/s  ({best:.3f} ms)")
