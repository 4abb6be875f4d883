"""Copy bandwidth vs working-set size (src + dst bytes): where L2 (126 MB)
stops holding the working set the rate falls to HBM's."""
import torch
torch.cuda.init()
for mb in [8, 16, 24, 32, 48, 64, 96, 128, 256, 1024]:
    n = mb * (1 << 20) // 2 // 2            # bf16 elements per buffer; src + dst = mb
    a = torch.randn(n, device="cuda").to(torch.bfloat16)
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    reps = 200 if mb <= 128 else 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"working set {mb:5d} MB: {2 * n * 2 / ms / 1e6:8.1f} GB/s  ({ms * 1e3:.1f} us per copy)")
