"""Time K1 alone on cfg5 (bf16 lin4 by default) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1905_05233_b200 as Wn
from paper_1905_05233_b200.algos import canonical_spec
name = sys.argv[1] if len(sys.argv) > 1 else "lin4"
dt = sys.argv[2] if len(sys.argv) > 2 else "bf16"
spec, m = canonical_spec(name)
a = Wn.WinoAlgo(spec, m)
tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
x = torch.relu(torch.randn(256, 512, 28, 28, device="cuda")).to(tdt)
for _ in range(3):
    V = Wn.wino_input_transform(x, a, pad=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    Wn.wino_input_transform(x, a, pad=1)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
nb = x.numel() * x.element_size() + V.numel() * V.element_size()
print(f"K1 {name} {dt} exp={os.environ.get('WINO_K1_EXP', '0')}: {us:.1f} us  {nb / us / 1e3:.0f} GB/s")
