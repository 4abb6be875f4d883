"""Compare the opt-in fused K3+K4 path against the staged one (run twice, WINO_FUSED=0/1)."""
import os, sys, subprocess, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import datagen, paper_1905_05233_b200 as W
from paper_1905_05233_b200.algos import canonical_spec
out = []
for name, dt, N, C, K, H, Wd in (('lin4', 'bf16', 3, 96, 272, 23, 19), ('sup1_6', 'fp16', 3, 96, 272, 23, 19),
                                 ('lin4', 'bf16', 8, 64, 512, 28, 28)):
    spec, m = canonical_spec(name)
    a = W.WinoAlgo(spec, m)
    x, w = datagen.layer(N, C, K, H, Wd, dt, seed=2)
    td = {'bf16': torch.bfloat16, 'fp16': torch.float16}[dt]
    y = W.wino_conv2d(torch.from_numpy(x).to(td).cuda(), torch.from_numpy(w).to(td).cuda(), a)
    torch.cuda.synchronize()
    out.append(y.float().cpu().numpy())
np.savez(sys.argv[1], *out)
"""
res = []
for fused in ("0", "1"):
    f = "/tmp/diag_fused_%s.npz" % fused
    env = dict(os.environ, WINO_FUSED=fused)
    r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300)
    print("fused", fused, "rc", r.returncode, r.stderr[-1500:])
    res.append(np.load(f))
for key in res[0].files:
    a, b = res[0][key], res[1][key]
    d = np.abs(a - b)
    bad = np.argwhere(d > 0)
    print(key, a.shape, "mismatch", len(bad), "of", a.size, "maxdiff", d.max(), "maxabs", np.abs(a).max())
    if len(bad):
        print("  first", bad[:8].tolist(), "nan in fused", np.isnan(b).sum())
        # which channels / rows are affected
        print("  channels", np.unique(bad[:, 1])[:40].tolist())
        print("  n", np.unique(bad[:, 0]).tolist(), "rows", np.unique(bad[:, 2])[:40].tolist())
a, b = res[0]["arr_1"], res[1]["arr_1"]
for k in range(0, 40):
    d = np.abs(a[:, k] - b[:, k])
    if d.max() == 0:
        continue
    match = [kk for kk in range(a.shape[1]) if np.array_equal(a[:, kk], b[:, k])]
    frac = (d > 0).mean()
    print("k", k, "frac wrong", round(float(frac), 3), "equals staged channel", match,
          "wrong n", np.unique(np.argwhere(d > 0)[:, 0]).tolist())
