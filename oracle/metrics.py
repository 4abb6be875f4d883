"""Error statistics (oracle component O9, metrics).  Test infrastructure only.

P:531 / P:548: "Euclidean error of Winograd convolution ... compared with the
direct convolution in fp64"; reading A12 adds the relative forms.  The 8-value
layout is SURVEY.md 8(b):

  [0] sum |y - yref|          [4] max_t ||y_t - yref_t|| / ||yref_t||
  [1] sum |yref|              [5] number of non-finite y
  [2] sum_t rel_t             [6] number of tiles
  [3] sum_t ||y_t - yref_t||  [7] number of elements

A tile t is one (n, k, m x m output block), clipped at ragged edges.  A
non-finite y makes its element error +inf.  rel_t = 0 when both norms are 0.
"""
import numpy as np


def stats8(y, yref, m):
    y = np.asarray(y, np.float64)
    yref = np.asarray(yref, np.float64)
    N, K, Ho, Wo = yref.shape
    th, tw = -(-Ho // m), -(-Wo // m)
    fin = np.isfinite(y)
    diff = np.where(fin, np.abs(y - yref), np.inf)
    pad = lambda a: np.pad(a, ((0, 0), (0, 0), (0, th * m - Ho), (0, tw * m - Wo)))
    tile = lambda a: pad(a).reshape(N, K, th, m, tw, m).sum(axis=(3, 5))
    with np.errstate(invalid="ignore", divide="ignore"):
        e2 = np.sqrt(tile(diff * diff))
        r2 = np.sqrt(tile(yref * yref))
        rel = np.where(e2 == 0, 0.0, e2 / np.where(r2 == 0, 0.0, r2))
    rel = np.where((r2 == 0) & (e2 > 0), np.inf, rel)
    return np.array([diff.sum(), np.abs(yref).sum(), rel.sum(), e2.sum(), rel.max(),
                     float((~fin).sum()), float(N * K * th * tw), float(y.size)])


def summary(s):
    return {"rel_l1": s[0] / s[1] if s[1] else float("nan"),
            "mean_rel": s[2] / s[6], "mean_euclid": s[3] / s[6],
            "max_rel": s[4], "nonfinite": int(s[5]), "tiles": int(s[6])}


def tile_rel_1d(y, yref):
    """Per-tile relative L2 error for batched 1D tiles (cfg 2)."""
    y = np.asarray(y, np.float64)
    yref = np.asarray(yref, np.float64)
    d = np.where(np.isfinite(y), y - yref, np.inf)
    e = np.sqrt((d * d).sum(axis=1))
    r = np.sqrt((yref * yref).sum(axis=1))
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(e == 0, 0.0, e / r)
