"""Time wino_conv2d_host_io (pinned host x -> device -> layer -> pinned host y) on cfg5,
as bench.py's e2e leg does; WINO_HOSTIO_CHUNKS picks the chunk count."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1905_05233_b200 as Wn
from paper_1905_05233_b200.algos import canonical_spec
spec, m = canonical_spec("lin4")
a = Wn.WinoAlgo(spec, m)
N, C, K, H, W = 256, 512, 512, 28, 28
x = torch.relu(torch.randn(N, C, H, W, device="cuda")).to(torch.bfloat16)
w = (torch.randn(K, C, 3, 3, device="cuda") * 0.02).to(torch.bfloat16)
y = torch.empty(N, K, H, W, dtype=torch.bfloat16, device="cuda")
ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(a, N, C, H, W, K, 1, "bf16"))
xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
xh.copy_(x.cpu())
yh = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
st = torch.cuda.current_stream()
for _ in range(2):
    Wn.wino_conv2d_host_io(xh, x, w, a, y, yh, ws, stream=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    Wn.wino_conv2d_host_io(xh, x, w, a, y, yh, ws, stream=st)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"chunks={os.environ.get('WINO_HOSTIO_CHUNKS', '8')}: {ms:.3f} ms  {2.0 * N * K * C * 9 * H * W / ms / 1e9:.1f} TFLOP/s")
