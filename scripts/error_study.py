"""Random-data error study on the GPU (Sec. 3.1, Figure 1):
floating-point error of Winograd convolution vs fp64 direct convolution for linear (Toom-Cook)
and superlinear point sets, 1D (kernel 3) and 2D (3x3), output tiles n = 2..8, as a function of
the multiplication ratio (1D mu/n, 2D mu^2/n^2).

* Inputs: "kernel and input values were chosen randomly from range (-1,1) with a normal
  distribution" (reading A14: N(0, 1/3) rejected outside (-1,1)); every trial draws its
  own kernel AND input tile, 5000 trials per (n, dtype), the same trials for every
  point set (paired).
* Error = mean per-trial Euclidean norm of (y - y_fp64), plus the mean relative error.
* 1D: K5 (wino_conv1d_tiles) in the paper's per-op rounding.
* bf16 paper-mode rows appear twice: round-to-nearest-even ("bf16") and truncation ("bf16-trunc",
  reading A10's switch: the paper calls bf16 "a truncated form of fp32", P:6); inputs are RNE
  bf16 values in both.
* 2D, paper mode: K7 (wino_conv2d_tiles_paper), per-op rounding as the paper simulated it.
* 2D, pipeline mode (the tensor-core layer): the whole layer (wino_conv2d) on batches of 64
  one-channel tiles against 64 kernels, keeping the diagonal (tile i, kernel i) pairs, so each
  trial still has its own kernel.
* Channel-sum boosters: paper-mode 2D tiles with C input channels summed sequentially vs
  pairwise, in the dtype vs in fp32 (mixed precision), against the pipeline layer.

    python scripts/error_study.py [--trials 5000] > profiles/error_study_r02.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POINTS = ["0", "-1", "1", "-1/2", "1/2", "2", "-2", "-1/4", "4"]
QUADS = ["a^2+1", "a^2+a+1", "a^2-a+1"]


def point_sets(n):
    """(family, moduli spec) for output size n: Toom-Cook, one quadratic (three choices), two quadratics."""
    out = [("lin", ",".join(POINTS[:n + 1] + ["inf"]))]
    if n >= 2:
        for q in QUADS:
            out.append((f"sup1[{q}]", ",".join(POINTS[:n - 1] + [q, "inf"])))
    if n >= 3:
        out.append(("sup2[a^2+1,a^2-2]", ",".join(POINTS[:n - 3] + ["a^2+1", "a^2-2", "inf"])))
    return out


def trunc_normal(rng, shape):
    import numpy as np
    out = rng.normal(0.0, 1.0 / 3.0, shape)
    bad = np.abs(out) >= 1
    while bad.any():
        out[bad] = rng.normal(0.0, 1.0 / 3.0, int(bad.sum()))
        bad = np.abs(out) >= 1
    return out


def trials2d(trials, n, seed, C=1):
    """Per-trial input tiles d[C][S][n+2][n+2] and kernels g[C][S][3][3] (fp64)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    return trunc_normal(rng, (C, trials, n + 2, n + 2)), trunc_normal(rng, (C, trials, 3, 3))


def direct2d(d, g):
    """fp64 valid correlation of every trial: [C][S][nx][nx] x [C][S][3][3] -> [S][n][n]."""
    import numpy as np
    nx = d.shape[-1]
    n = nx - 2
    y = np.zeros((d.shape[1], n, n))
    for p in range(3):
        for q in range(3):
            y += (g[:, :, p, q][:, :, None, None] * d[:, :, p:p + n, q:q + n]).sum(0)
    return y


def errs(y, ref):
    """(mean per-trial Euclidean error, mean per-trial relative error, non-finite count)."""
    import numpy as np
    y = y.reshape(y.shape[0], -1)
    ref = ref.reshape(ref.shape[0], -1)
    d = np.where(np.isfinite(y), y - ref, np.inf)
    e = np.sqrt((d * d).sum(1))
    r = np.sqrt((ref * ref).sum(1))
    return float(e.mean()), float(np.mean(np.where(r > 0, e / np.maximum(r, 1e-300), 0.0))), int((~np.isfinite(y)).sum())


def pipeline_diag(Wn, algo, d, g, td):
    """The tensor-core layer on one-channel tiles, 64 tiles x 64 kernels per call;
    y[i] = output of (tile i, kernel i)."""
    import numpy as np
    import torch
    S = d.shape[1]
    out = []
    for s0 in range(0, S, 64):
        xb = torch.from_numpy(np.ascontiguousarray(d[0, s0:s0 + 64][:, None])).to(td).cuda()
        wb = torch.from_numpy(np.ascontiguousarray(g[0, s0:s0 + 64][:, None])).to(td).cuda()
        y = Wn.wino_conv2d(xb, wb, algo, pad=0)                       # [b][b][n][n]
        idx = torch.arange(xb.shape[0], device=y.device)
        out.append(y[idx, idx].double().cpu().numpy())
    return np.concatenate(out)


def run(trials, dtypes=("fp32", "fp16", "bf16"), ns=range(2, 9), seed=0, pipeline=True):
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    td = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
    rows = []
    for n in ns:
        rng = np.random.default_rng(seed + n)
        x1, h1 = trunc_normal(rng, (trials, n + 2)), trunc_normal(rng, (trials, 3))
        d2, g2 = trials2d(trials, n, seed + 100 + n)
        for dt in dtypes:
            x1d, h1d = datagen.to_dtype_values(x1, dt), datagen.to_dtype_values(h1, dt)
            ref1 = np.stack([(x1d[:, i:i + 3] * h1d).sum(1) for i in range(n)], 1)   # fp64 direct correlation
            d2d, g2d = datagen.to_dtype_values(d2, dt), datagen.to_dtype_values(g2, dt)
            ref2 = direct2d(d2d, g2d)
            dt_d = torch.from_numpy(d2d).to(td[dt]).cuda()
            dt_g = torch.from_numpy(g2d).to(td[dt]).cuda()
            for fam, spec in point_sets(n):
                algo = Wn.WinoAlgo(spec, n)
                y1 = Wn.wino_conv1d_tiles(torch.from_numpy(x1d).to(td[dt]).cuda(),
                                          torch.from_numpy(h1d).to(td[dt]).cuda(), algo, per_op_rounding=True)
                e, r, nf = errs(y1.double().cpu().numpy(), ref1)
                rows.append({"dim": 1, "mode": "paper", "family": fam, "spec": spec, "n": n, "mu": algo.mu,
                             "dtype": dt, "ratio": algo.mu / n, "mean_euclid": e, "mean_rel": r, "nonfinite": nf})
                y2 = Wn.wino_conv2d_tiles_paper(dt_d, dt_g, algo)
                e, r, nf = errs(y2.double().cpu().numpy(), ref2)
                rows.append({"dim": 2, "mode": "paper", "family": fam, "spec": spec, "n": n, "mu": algo.mu,
                             "dtype": dt, "ratio": algo.mu ** 2 / n ** 2, "mean_euclid": e, "mean_rel": r,
                             "nonfinite": nf})
                if dt == "bf16":
                    # the paper's "truncated form of fp32" read as a rounding mode (reading A10's switch)
                    y1t = Wn.wino_conv1d_tiles(torch.from_numpy(x1d).to(td[dt]).cuda(),
                                               torch.from_numpy(h1d).to(td[dt]).cuda(), algo, per_op_rounding=True,
                                               bf16_mode="trunc")
                    e, r, nf = errs(y1t.double().cpu().numpy(), ref1)
                    rows.append({"dim": 1, "mode": "paper", "family": fam, "spec": spec, "n": n, "mu": algo.mu,
                                 "dtype": "bf16-trunc", "ratio": algo.mu / n, "mean_euclid": e, "mean_rel": r,
                                 "nonfinite": nf})
                    y2t = Wn.wino_conv2d_tiles_paper(dt_d, dt_g, algo, bf16_mode="trunc")
                    e, r, nf = errs(y2t.double().cpu().numpy(), ref2)
                    rows.append({"dim": 2, "mode": "paper", "family": fam, "spec": spec, "n": n, "mu": algo.mu,
                                 "dtype": "bf16-trunc", "ratio": algo.mu ** 2 / n ** 2, "mean_euclid": e,
                                 "mean_rel": r, "nonfinite": nf})
                if pipeline:
                    e, r, nf = errs(pipeline_diag(Wn, algo, d2d, g2d, td[dt]), ref2)
                    rows.append({"dim": 2, "mode": "pipeline", "family": fam, "spec": spec, "n": n, "mu": algo.mu,
                                 "dtype": dt, "ratio": algo.mu ** 2 / n ** 2, "mean_euclid": e, "mean_rel": r,
                                 "nonfinite": nf})
    return rows


def boosters(trials=2000, Cs=(16, 64, 256), names=("lin4", "sup1_6", "lin6"), dtypes=("fp16", "bf16"), seed=7):
    """Channel-sum variants of P:611 on paper-mode 2D tiles with C channels."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    td = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
    rows = []
    for name in names:
        spec, m = canonical_spec(name)
        algo = Wn.WinoAlgo(spec, m)
        for C in Cs:
            d, g = trials2d(trials, m, seed + C, C=C)
            for dt in dtypes:
                dd, gd = datagen.to_dtype_values(d, dt), datagen.to_dtype_values(g, dt)
                ref = direct2d(dd, gd)
                tdd, tgd = torch.from_numpy(dd).to(td[dt]).cuda(), torch.from_numpy(gd).to(td[dt]).cuda()
                for csum in ("sequential", "pairwise"):
                    for acc in ("dtype", "fp32"):
                        e, r, nf = errs(Wn.wino_conv2d_tiles_paper(tdd, tgd, algo, csum, acc).double().cpu().numpy(), ref)
                        rows.append({"algo": name, "C": C, "dtype": dt, "mode": f"paper/{csum}/{acc}",
                                     "mean_euclid": e, "mean_rel": r, "nonfinite": nf})
    return rows


def pareto(rows):
    """Best (lowest mean Euclidean error) point set per (dim, mode, dtype, ratio), and the Pareto front."""
    out = {}
    for dim, mode in ((1, "paper"), (2, "paper"), (2, "pipeline")):
        for dt in sorted({r["dtype"] for r in rows}):
            rs = sorted([r for r in rows if r["dim"] == dim and r["mode"] == mode and r["dtype"] == dt],
                        key=lambda r: (r["ratio"], r["mean_euclid"]))
            if not rs:
                continue
            front, best = [], float("inf")
            for r in rs:
                if r["mean_euclid"] < best:
                    best = r["mean_euclid"]
                    front.append({k: r[k] for k in ("family", "n", "mu", "ratio", "mean_euclid")})
            out[f"{dim}d/{mode}/{dt}"] = front[::-1]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=5000)
    a = ap.parse_args()
    rows = run(a.trials)
    print(json.dumps({"trials": a.trials, "inputs": "N(0,1/3) rejected outside (-1,1), fresh kernel and tile per "
                                                    "trial (P:531, reading A14, SPEC S:429)",
                      "rows": rows, "pareto": pareto(rows), "boosters": boosters()}, indent=1))


if __name__ == "__main__":
    main()
