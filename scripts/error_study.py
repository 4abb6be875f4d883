"""Random-data error study on the GPU (Sec. 3.1, Figure 1):
floating-point error of Winograd convolution vs fp64 direct convolution for linear (Toom-Cook)
and superlinear point sets, 1D (kernel 3) and 2D (3x3), output tiles n = 2..8, as a function of
the multiplication ratio (1D mu/n, 2D mu^2/n^2).  Inputs drawn "randomly from range (-1,1) with a
normal distribution" (reading A14: N(0, 1/3) rejected outside (-1,1)), 5000 paired tiles per
(n, dtype) shared by every point set.  Error = mean per-tile Euclidean norm of (y - y_fp64),
plus the mean per-tile relative error.  1D runs K5 (wino_conv1d_tiles, paper per-op rounding);
2D runs the whole layer (wino_conv2d) on N tiles of one channel (pad 0, one output tile each).

    python scripts/error_study.py [--trials 5000] > profiles/error_study_r01.json
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


def run(trials, dtypes=("fp32", "fp16", "bf16"), ns=range(2, 9), seed=0):
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    td = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
    rows = []
    for n in ns:
        rng = np.random.default_rng(seed + n)
        x1, h1 = trunc_normal(rng, (trials, n + 2)), trunc_normal(rng, (trials, 3))
        x2, w2 = trunc_normal(rng, (trials, 1, n + 2, n + 2)), trunc_normal(rng, (1, 1, 3, 3))
        for dt in dtypes:
            x1d, h1d = datagen.to_dtype_values(x1, dt), datagen.to_dtype_values(h1, dt)
            ref1 = np.stack([(x1d[:, i:i + 3] * h1d).sum(1) for i in range(n)], 1)   # fp64 direct correlation
            x2d, w2d = datagen.to_dtype_values(x2, dt), datagen.to_dtype_values(w2, dt)
            xt = torch.from_numpy(x2d).to(td[dt]).cuda()
            wt = torch.from_numpy(w2d).to(td[dt]).cuda()
            ref2 = Wn.wino_direct_conv2d_f64(xt, wt, 0)
            for fam, spec in point_sets(n):
                algo = Wn.WinoAlgo(spec, n)
                # 1D: K5 in the paper's per-op rounding
                y1 = Wn.wino_conv1d_tiles(torch.from_numpy(x1d).to(td[dt]).cuda(),
                                          torch.from_numpy(h1d).to(td[dt]).cuda(), algo, per_op_rounding=True)
                y1 = y1.double().cpu().numpy()
                d = np.where(np.isfinite(y1), y1 - ref1, np.inf)
                e1 = np.sqrt((d * d).sum(1))
                r1 = np.sqrt((ref1 * ref1).sum(1))
                rows.append({"dim": 1, "family": fam, "spec": spec, "n": n, "mu": algo.mu, "dtype": dt,
                             "ratio": algo.mu / n, "mean_euclid": float(e1.mean()),
                             "mean_rel": float(np.mean(np.where(r1 > 0, e1 / np.maximum(r1, 1e-300), 0.0))),
                             "nonfinite": int((~np.isfinite(y1)).sum())})
                # 2D: the whole layer on one-channel single tiles
                y2 = Wn.wino_conv2d(xt, wt, algo, pad=0)
                s = Wn.summary(Wn.wino_error_stats(y2, ref2, n).cpu())
                rows.append({"dim": 2, "family": fam, "spec": spec, "n": n, "mu": algo.mu, "dtype": dt,
                             "ratio": algo.mu ** 2 / n ** 2, "mean_euclid": s["mean_euclid"],
                             "mean_rel": s["mean_rel"], "nonfinite": s["nonfinite"]})
    return rows


def pareto(rows):
    """Best (lowest mean Euclidean error) point set per (dim, dtype, ratio), and the Pareto front."""
    out = {}
    for dim in (1, 2):
        for dt in sorted({r["dtype"] for r in rows}):
            rs = sorted([r for r in rows if r["dim"] == dim and r["dtype"] == dt], key=lambda r: (r["ratio"], r["mean_euclid"]))
            front, best = [], float("inf")
            for r in rs:
                if r["mean_euclid"] < best:
                    best = r["mean_euclid"]
                    front.append({k: r[k] for k in ("family", "n", "mu", "ratio", "mean_euclid")})
            out[f"{dim}d/{dt}"] = front[::-1]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=5000)
    a = ap.parse_args()
    rows = run(a.trials)
    print(json.dumps({"trials": a.trials, "inputs": "N(0,1/3) rejected outside (-1,1) (P:531, reading A14)",
                      "rows": rows, "pareto": pareto(rows)}, indent=1))


if __name__ == "__main__":
    main()
