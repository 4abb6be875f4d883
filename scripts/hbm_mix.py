"""HBM bandwidth by access mix on this B200: pure write (memset), pure read
(sum), copy (read+write), and a 1:2 read:write mix like K3's (V read, fp32 M
written).  CUDA events, 2 GiB buffers (>> L2), best of 5."""
import torch

def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return nbytes / best / 1e9

n = 1 << 29   # 2 GiB of fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
h = torch.empty(n // 2, device="cuda")
print("write (fill)      %.0f GB/s" % bw(lambda: a.fill_(1.0), 4 * n))
print("read (sum)        %.0f GB/s" % bw(lambda: a.sum(), 4 * n))
print("copy (r+w)        %.0f GB/s" % bw(lambda: b.copy_(a), 8 * n))
print("r:w = 1:2 (h->a,b) %.0f GB/s" % bw(lambda: (a[: n // 2].copy_(h), a[n // 2:].copy_(h)), 4 * (n // 2) * 4))
