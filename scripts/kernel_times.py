"""Per-kernel CUDA-event times (K2, K1, K3, K4) and the whole step of one cfg5-shaped
layer, for A/B comparisons of kernel variants (environment switches such as
WINO_PAIR=0; KT_M_STORE=dtype selects M in the 16-bit dtype).  Random synthetic
inputs (torch), no oracle.

    python scripts/kernel_times.py [algo] [dtype] [N] [C] [K] [H]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_05233_b200 as Wn
from paper_1905_05233_b200.algos import canonical_spec

name = sys.argv[1] if len(sys.argv) > 1 else "lin4"
dt = sys.argv[2] if len(sys.argv) > 2 else "bf16"
N, C, K, H = (int(v) for v in (sys.argv[3:7] + ["256", "512", "512", "28"][len(sys.argv[3:7]):]))
spec, m = canonical_spec(name)
a = Wn.WinoAlgo(spec, m)
if os.environ.get("KT_M_STORE", "fp32") == "dtype":   # M3: M stored in the 16-bit dtype
    a.set_m_storage("dtype")
tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
torch.manual_seed(0)
x = torch.relu(torch.randn(N, C, H, H, device="cuda")).to(tdt)
w = (torch.randn(K, C, 3, 3, device="cuda") * (2.0 / (9 * C)) ** 0.5).to(tdt)
y = torch.empty((N, K, H, H), dtype=tdt, device="cuda")
ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(a, N, C, H, H, K, 1, dt, "nchw"))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
kern = bench.per_kernel_times(a, x, w, y, ws, st, N, C, K, H, H, dt, 20)
with torch.cuda.stream(st):
    for _ in range(3):
        Wn.wino_conv2d(x, w, a, out=y, workspace=ws, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        Wn.wino_conv2d(x, w, a, out=y, workspace=ws, stream=st)
    e1.record(st)
torch.cuda.synchronize()
out = {"algo": name, "dtype": dt, "shape": [N, C, K, H], "env": {k: v for k, v in os.environ.items() if k.startswith(("WINO_", "KT_"))},
       "step_us_eager": e0.elapsed_time(e1) / 50 * 1e3, "kernels_us": {k: v * 1e3 for k, v in kern.items()}}
print(json.dumps(out))
