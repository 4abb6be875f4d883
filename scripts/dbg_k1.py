"""Run K1 alone on shapes that reach each staging path; report failures."""
import sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cases = [("bf16", 28, 28, "lin4"), ("fp16", 28, 28, "lin4"), ("bf16", 32, 32, "lin4"), ("fp32", 32, 32, "lin4"),
         ("fp32", 28, 28, "lin4"), ("bf16", 14, 14, "lin2"), ("bf16", 56, 56, "lin6")]
if len(sys.argv) > 1:
    import torch, numpy as np
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    dt, H, Wd, name = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    spec, m = canonical_spec(name)
    a = Wn.WinoAlgo(spec, m)
    tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
    x = torch.randn(2, 64, H, Wd).to(tdt).cuda()
    V = Wn.wino_input_transform(x, a, pad=1)
    torch.cuda.synchronize()
    print("ok", dt, H, Wd, name, float(V[0].float().abs().sum()))
else:
    for c in cases:
        r = subprocess.run([sys.executable, __file__] + [str(v) for v in c], capture_output=True, text=True,
                           env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
        print(c, "rc", r.returncode, (r.stdout + r.stderr).strip().splitlines()[-1:] )
