"""Pins for WHERE the emulated-precision oracle rounds (oracle/precision.py).

The trend pins in test_oracle_precision.py hold for any reasonable rounding
model; these hand-derived cases (tests/golden/rounding_points.json, each with
its arithmetic written out) fail as soon as a rounding point is moved, added or
dropped:

* PAPER mode: every product and partial sum is cast
  to the dtype -- a single-cast accumulation gives 2050 / 258 instead of
  2048 / 256 on the dot examples, end to end through po_matmul, paper_conv1d
  and paper_conv2d_tiles (including the channel sum in the Winograd domain).
* PIPELINE mode (reading R1): V = rd(B^T d B) and U = rd(G g G^T) are
  rounded once each, M is not, y is rounded once.  One single-tile,
  single-channel F(2x2, 3x3) layer per (dtype, tensor) has exactly one tie in V
  (resp. U); the expected y is the direct correlation plus A^T (U (.) Delta) A
  for that one rounding step, then one cast of the result.
Expected values use Fractions and the library casts of torch, never the oracle.
"""
import json
import os
from fractions import Fraction as Fr
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import precision as P
from oracle import transforms as T

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rounding_points.json")
TDT = {"fp16": torch.float16, "bf16": torch.bfloat16}


def _gold():
    with open(GOLD) as f:
        return json.load(f)


def _cast(v, dtype):
    """One library cast (torch, RNE) of an exactly representable-in-fp32 value."""
    return float(torch.tensor(float(v), dtype=torch.float32).to(TDT[dtype]).float())


def _direct(d, g):
    """Valid 2D cross-correlation of a 4x4 tile with a 3x3 kernel (reading A5)."""
    return [[sum(Fr(g[p][q]) * Fr(d[i + p][j + q]) for p in range(3) for q in range(3)) for j in range(2)]
            for i in range(2)]


# --------------------------------------------------------------------------- paper mode


@pytest.mark.parametrize("case", _gold()["paper_dot"], ids=lambda c: c["dtype"])
def test_paper_dot_casts_every_partial_sum(case):
    dt = case["dtype"]
    u = np.array([case["u"]], np.float32)
    v = np.array(case["v"], np.float32)[:, None]
    got = P.po_matmul(u, v, dt)[0, 0]
    assert got == case["per_op"]
    # the case discriminates: one cast of the exact sum is the other value
    assert _cast(sum(a * b for a, b in zip(case["u"], case["v"])), dt) == case["single_cast"] != case["per_op"]


def _sum_algo():
    """A 1-point 'algorithm' (G = [1 0 0], B^T = [1 1 1], A^T = [1]): u = h_0,
    v = x_0 + x_1 + x_2, y = u v -- the paper-mode pipeline reduced to one dot."""
    return SimpleNamespace(G=[[1, 0, 0]], BT=[[1, 1, 1]], AT=[[1]], n_o=1, n_x=3, mu=1)


@pytest.mark.parametrize("case", _gold()["paper_dot"], ids=lambda c: c["dtype"])
def test_paper_conv1d_rounds_per_op(case):
    dt = case["dtype"]
    x = np.array([case["v"]], np.float32)                     # one tile, n_x = 3
    h = np.array([[1, 0, 0]], np.float32)
    assert P.paper_conv1d(_sum_algo(), x, h, dt)[0, 0] == case["per_op"]


@pytest.mark.parametrize("case", _gold()["paper_dot"], ids=lambda c: c["dtype"])
def test_paper_conv2d_tiles_rounds_per_op(case):
    """Row stage, column stage and the channel sum are each cast per op."""
    dt = case["dtype"]
    big, one = float(case["v"][0]), float(case["v"][1])
    ts = _sum_algo()
    # one channel: the row stage sums column 0 = [big, 1, 1] per op
    d = np.zeros((1, 1, 3, 3), np.float32)
    d[0, 0, :, 0] = [big, one, one]
    g = np.zeros((1, 1, 3, 3), np.float32)
    g[0, 0, 0, 0] = 1
    assert P.paper_conv2d_tiles(ts, d, g, dt)[0, 0, 0] == case["per_op"]
    # column stage: row 0 = [big, 1, 1]
    d2 = np.zeros((1, 1, 3, 3), np.float32)
    d2[0, 0, 0, :] = [big, one, one]
    assert P.paper_conv2d_tiles(ts, d2, g, dt)[0, 0, 0] == case["per_op"]
    # channel sum in the Winograd domain: three channels carrying big, 1, 1
    d3 = np.zeros((3, 1, 3, 3), np.float32)
    d3[:, 0, 0, 0] = [big, one, one]
    g3 = np.zeros((3, 1, 3, 3), np.float32)
    g3[:, 0, 0, 0] = 1
    assert P.paper_conv2d_tiles(ts, d3, g3, dt)[0, 0, 0] == case["per_op"]


# --------------------------------------------------------------------------- pipeline mode


def _lin2():
    g = _gold()["lin2_matrices"]
    return [[Fr(v) for v in r] for r in g["G"]], [[Fr(v) for v in r] for r in g["BT"]], \
        [[Fr(v) for v in r] for r in g["AT"]]


def test_lin2_matrices_are_the_generated_ones():
    """The literal matrices of the golden file are those the oracle generates for
    {0, -1, 1, inf} (pinned against the paper elsewhere); this keeps the hand
    derivations below about the algorithm the oracle actually runs."""
    G, BT, AT = _lin2()
    mods, m = T.canonical("lin2")
    ts = T.make_transforms(mods, m)
    assert ts.G == G and ts.BT == BT and ts.AT == AT


def _expected(case, tensor):
    G, BT, AT = _lin2()
    d, g = case["d"], case["g"]
    a, b = case["point"]
    y = _direct(d, g)
    if tensor == "V":
        delta = Fr(case["V_rounded"]) - Fr(case["V_exact"])
        other = Fr(case["U_at_point"])
    else:
        delta = Fr(case["U_rounded"]) - Fr(case["U_exact"])
        other = Fr(case["V_at_point"])
    # A^T (U (.) V) A changes by other * delta * AT[:, a] AT[:, b]^T
    return [[_cast(y[i][j] + other * delta * AT[i][a] * AT[j][b], case["dtype"]) for j in range(2)]
            for i in range(2)], [[_cast(y[i][j], case["dtype"]) for j in range(2)] for i in range(2)]


def _check_hand_arithmetic(case, tensor):
    """Re-derive the tie stated in the golden file from the literal matrices."""
    G, BT, AT = _lin2()
    a, b = case["point"]
    d = [[Fr(v) for v in r] for r in case["d"]]
    g = [[Fr(v) for v in r] for r in case["g"]]
    V = [[sum(BT[p][i] * d[i][j] * BT[q][j] for i in range(4) for j in range(4)) for q in range(4)] for p in range(4)]
    U = [[sum(G[p][i] * g[i][j] * G[q][j] for i in range(3) for j in range(3)) for q in range(4)] for p in range(4)]
    dt = case["dtype"]
    rV = [[_cast(v, dt) for v in r] for r in V]
    rU = [[_cast(v, dt) for v in r] for r in U]
    changed_V = [(p, q) for p in range(4) for q in range(4) if rV[p][q] != V[p][q]]
    changed_U = [(p, q) for p in range(4) for q in range(4) if rU[p][q] != U[p][q]]
    if tensor == "V":
        assert changed_V == [(a, b)] and changed_U == []
        assert V[a][b] == Fr(case["V_exact"]) and rV[a][b] == Fr(case["V_rounded"]) and U[a][b] == case["U_at_point"]
    else:
        assert changed_U == [(a, b)] and changed_V == []
        assert U[a][b] == case["U_exact"] and rU[a][b] == case["U_rounded"] and V[a][b] == Fr(case["V_at_point"])


@pytest.mark.parametrize("tensor", ["V", "U"])
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_pipeline_rounds_stored_tensors_once(tensor, dtype):
    case = next(c for c in _gold()["pipeline_" + tensor] if c["dtype"] == dtype)
    _check_hand_arithmetic(case, tensor)
    want, unrounded_model = _expected(case, tensor)
    assert want != unrounded_model                      # the case discriminates
    mods, m = T.canonical("lin2")
    ts = T.make_transforms(mods, m)
    x = np.array(case["d"], np.float32)[None, None]     # [N=1, C=1, 4, 4], pad 0 -> one 2x2 tile
    w = np.array(case["g"], np.float32)[None, None]
    y = P.pipeline_conv2d(ts, x, w, dtype, pad=0)
    assert y[0, 0].tolist() == want


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_pipeline_accumulates_M_in_fp32(dtype):
    """M = sum_c U V is not rounded to the dtype: three channels carry big, 1
    and 1 (big = 256 in bf16, 2048 in fp16) to the same output; the exact
    big + 2 is a dtype value, while a dtype-rounded running sum loses each 1
    (big + 1 is a tie that rounds to big)."""
    mods, m = T.canonical("lin2")
    ts = T.make_transforms(mods, m)
    big = 256.0 if dtype == "bf16" else 2048.0
    x = np.zeros((1, 3, 4, 4), np.float32)
    x[0, :, 1, 1] = [big, 1.0, 1.0]
    w = np.zeros((1, 3, 3, 3), np.float32)
    w[0, :, 1, 1] = 1.0      # centre tap: y[i][j] = sum_c x[c][i+1][j+1]
    y = P.pipeline_conv2d(ts, x, w, dtype, pad=0)
    assert y[0, 0].tolist() == [[big + 2, 0.0], [0.0, 0.0]]


# --------------------------------------------------------------------------- channel-sum boosters


@pytest.mark.parametrize("case", _gold()["channel_sum"]["cases"], ids=lambda c: f'{c["dtype"]}-C{len(c["P"])}')
@pytest.mark.parametrize("csum", ["sequential", "pairwise"])
@pytest.mark.parametrize("acc", ["dtype", "fp32"])
def test_paper_conv2d_tiles_channel_sum_variants(case, csum, acc):
    """The channel sum of the paper-mode 2D tiles, sequential vs pairwise and
    dtype vs fp32 (mixed precision) accumulation: channel c carries the product
    P_c at the single Winograd point of the 1-point algorithm."""
    dt = case["dtype"]
    C = len(case["P"])
    d = np.zeros((C, 1, 3, 3), np.float32)
    d[:, 0, 0, 0] = case["P"]
    g = np.zeros((C, 1, 3, 3), np.float32)
    g[:, 0, 0, 0] = 1
    got = P.paper_conv2d_tiles(_sum_algo(), d, g, dt, csum=csum, acc=acc)[0, 0, 0]
    assert got == case[f"{csum}_{acc}"]


def test_pairwise_sum_tree_shape():
    """pairwise_sum's tree: h = the largest power of two below n (records the
    association with strings)."""
    add = lambda a, b: f"({a}+{b})"   # noqa: E731
    assert P.pairwise_sum(list("abcde"), add) == "(((a+b)+(c+d))+e)"
    assert P.pairwise_sum(list("abcdef"), add) == "(((a+b)+(c+d))+(e+f))"
    assert P.pairwise_sum(list("abcdefg"), add) == "(((a+b)+(c+d))+((e+f)+g))"
    assert P.pairwise_sum(list("a"), add) == "a"


# --------------------------------------------------------------------------- M storage (reading M3)


@pytest.mark.parametrize("case", _gold()["pipeline_M_dtype"]["cases"], ids=lambda c: c["dtype"])
def test_pipeline_m_store_dtype_rounds_M_once(case):
    """m_store="dtype": the fp32 channel sum M is rounded once to the dtype
    before the output transform.  The golden file states M (exact), its ties
    and both models' y; here M is recomputed with Fractions from the literal
    lin2 matrices, the stated ties are checked against a torch cast, and the
    oracle must give y_fp32_M with m_store="fp32" and y_dtype_M with "dtype"."""
    G, BT, AT = _lin2()
    dt, big = case["dtype"], case["big"]
    d = [[[Fr(0)] * 4 for _ in range(4)] for _ in range(2)]
    g = [[[Fr(0)] * 3 for _ in range(3)] for _ in range(2)]
    d[0][1][1], g[0][1][1] = Fr(big), Fr(1)
    (a, b), (i1, j1) = case["pos1"], case["tap1"]
    d[1][a][b], g[1][i1][j1] = Fr(1), Fr(1)
    M = [[sum(sum(G[p][i] * g[c][i][j] * G[q][j] for i in range(3) for j in range(3)) *
              sum(BT[p][i] * d[c][i][j] * BT[q][j] for i in range(4) for j in range(4)) for c in range(2))
          for q in range(4)] for p in range(4)]
    assert [[str(v) for v in r] for r in M] == case["M_exact"]
    rM = [[Fr(_cast(v, dt)) for v in r] for r in M]
    changed = {str(M[p][q]): str(rM[p][q]) for p in range(4) for q in range(4) if rM[p][q] != M[p][q]}
    assert changed == case["ties"]
    y_hand = [[_cast(sum(AT[i][p] * rM[p][q] * AT[j][q] for p in range(4) for q in range(4)), dt)
               for j in range(2)] for i in range(2)]
    assert y_hand == case["y_dtype_M"] and y_hand != case["y_fp32_M"]
    mods, m = T.canonical("lin2")
    ts = T.make_transforms(mods, m)
    x = np.zeros((1, 2, 4, 4), np.float32)
    w = np.zeros((1, 2, 3, 3), np.float32)
    x[0, 0, 1, 1], w[0, 0, 1, 1] = big, 1.0
    x[0, 1, a, b], w[0, 1, i1, j1] = 1.0, 1.0
    assert P.pipeline_conv2d(ts, x, w, dt, pad=0)[0, 0].tolist() == case["y_fp32_M"]
    assert P.pipeline_conv2d(ts, x, w, dt, pad=0, m_store="dtype")[0, 0].tolist() == case["y_dtype_M"]


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_m_store_dtype_bound_holds(dtype):
    """The M3 elementwise bound covers the dtype-M oracle on a random layer, and
    the plain R1 bound does not need to (the extra u_d S term is what M adds)."""
    from oracle import conv as CV
    import datagen
    mods, m = T.canonical("lin4")
    ts = T.make_transforms(mods, m)
    x, w = datagen.layer(1, 16, 8, 12, 12, dtype, seed=3)
    yref = CV.direct_conv2d_f64(x, w, pad=1)
    y = P.pipeline_conv2d(ts, x, w, dtype, m_store="dtype")
    bd = P.elementwise_bound(ts, x, w, dtype, yref, m_store="dtype")
    assert np.all(np.abs(y - yref) <= bd)
