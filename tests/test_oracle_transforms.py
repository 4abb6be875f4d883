"""Pins for oracle/transforms.py (O2-O6) against what the paper fixes:

* the printed worked example, golden/worked_example.json;
* the textbook special case: Toom-Cook point sets reproduce the standard Lavin-Gray
  F(2,3) and F(4,3) matrices (the paper's [Lavin16]) up to a per-point row
  scaling g_i b_i a_i = 1, the standard matrices being exact on their own;
* the printed multiplication counts (Table 1),
  golden/ratios.json;
* brute force: exact-rational Winograd equals direct correlation (CRT, Eq. 1).
"""
import itertools
import json
import os
import random
from fractions import Fraction as Fr

import pytest

from oracle import conv as CV
from oracle import exact as X
from oracle import transforms as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _ev(expr, b, c):
    return Fr(eval(expr, {"__builtins__": {}}, {"b": Fr(b), "c": Fr(c)}))


def _mat(entry, b, c):
    return [[_ev(e, b, c) for e in row] for row in entry["rows"]]


# irreducible a^2 + b a + c over Q (non-square discriminant b^2 - 4c)
BC = [(0, 1), (1, 1), (-1, 1), (0, 2), (1, 3), (2, 3), (0, -2), (3, 5)]


@pytest.mark.parametrize("b,c", BC)
def test_worked_example_general_bc(b, c):
    g = _gold("worked_example.json")
    quad = T.poly_mod((Fr(c), Fr(b), Fr(1)))
    mods = [T.point(0), quad, T.inf()]
    sp = [Fr(0), Fr(1), T.INF]                                   # P:243 points 0, 1
    Gtc, Atc, Btc = T.toom_cook_subsolver(sp, 2)
    assert Gtc == _mat(g["G_TC"], b, c)
    assert Atc == _mat(g["A_TC"], b, c)
    assert Btc == _mat(g["B_TC"], b, c)
    assert T._residue_map(quad.poly, 3) == _mat(g["Gprime"], b, c)
    assert T._residue_map(quad.poly, 4) == _mat(g["Aprime"], b, c)   # printed A' (4 columns)
    G, A = T.algorithm1(mods, 2, 3, sp)
    assert G == _mat(g["G_W"], b, c)
    assert G[1:4] == _mat(g["G_2"], b, c)
    # reading A1: only the first n_o = 2 columns of the printed A_2 / A^W
    # the pseudo-point row is [0 ... 0 1] of length n_o (Algorithm 1)
    assert A[:4] == [r[:2] for r in _mat(g["A_W"], b, c)[:4]]
    assert A[4] == [0, 1]
    assert A[1:4] == [r[:2] for r in _mat(g["A_2"], b, c)]
    B, C, E = T.algorithm2(mods, 2, 3, sp, return_parts=True)
    assert C == _mat(g["C"], b, c)
    assert [r[1:] for r in C[1:]] == _mat(g["C_2"], b, c)
    # the generated algorithm is exact for every (b, c) (reading A2: extended Euclid)
    ts = T.make_transforms(mods, 2, 3, sp)
    rng = random.Random(b * 31 + c)
    for _ in range(20):
        h = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(3)]
        x = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(4)]
        assert CV.winograd_1d_exact(ts, h, x) == CV.direct_corr_1d(h, x)


def test_worked_example_printed_E_BW_at_b0_c1():
    """P:445-494 printed N_i, E, B^W hold at (b, c) = (0, 1) (reading A2)."""
    g = _gold("worked_example.json")
    b, c = 0, 1
    quad = T.poly_mod((Fr(c), Fr(b), Fr(1)))
    mods = [T.point(0), quad, T.inf()]
    sp = [Fr(0), Fr(1), T.INF]
    M = X.prod([m.poly for m in mods[:2]])
    N1, _ = X.ext_euclid(mods[0].poly, X.divmod_(M, mods[0].poly)[0])
    N2, _ = X.ext_euclid(quad.poly, X.divmod_(M, quad.poly)[0])
    assert list(N1) == [Fr(v) for v in g["N_1"]["poly"]]
    assert list(N2) == [Fr(v) for v in g["N_2"]["poly"]]
    B, C, E = T.algorithm2(mods, 2, 3, sp, return_parts=True)
    assert E == _mat(g["E"], b, c)
    assert B == _mat(g["B_W"], b, c)


def test_printed_bw_not_exact_for_other_bc():
    """The printed B^W is not a valid input transform for a^2+a+1
    (reading A2) -- guards against 'fixing' the generator to match it."""
    g = _gold("worked_example.json")
    b, c = 1, 1
    quad = T.poly_mod((Fr(c), Fr(b), Fr(1)))
    ts = T.make_transforms([T.point(0), quad, T.inf()], 2, 3, [Fr(0), Fr(1), T.INF])
    printed = _mat(g["B_W"], b, c)
    assert printed != ts.B
    ts.B = printed
    rng = random.Random(5)
    bad = 0
    for _ in range(10):
        h = [Fr(rng.randint(-9, 9)) for _ in range(3)]
        x = [Fr(rng.randint(-9, 9)) for _ in range(4)]
        bad += CV.winograd_1d_exact(ts, h, x) != CV.direct_corr_1d(h, x)
    assert bad > 0


# ------------------------------------------------------------------ textbook special case
# Standard (Lavin-Gray) Winograd minimal filtering matrices, correlation form
# Y = A^T [(G g) (.) (B^T d)], points (0, 1, -1, inf) and (0, 1, -1, 2, -2, inf).
LAVIN_F23 = dict(
    BT=[[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, 1, 0, -1]],
    G=[[1, 0, 0], ["1/2", "1/2", "1/2"], ["1/2", "-1/2", "1/2"], [0, 0, 1]],
    AT=[[1, 1, 1, 0], [0, 1, -1, -1]],
    points="0,1,-1,inf", m=2)
LAVIN_F43 = dict(
    BT=[[4, 0, -5, 0, 1, 0], [0, -4, -4, 1, 1, 0], [0, 4, -4, -1, 1, 0],
        [0, -2, -1, 2, 1, 0], [0, 2, -1, -2, 1, 0], [0, 4, 0, -5, 0, 1]],
    G=[["1/4", 0, 0], ["-1/6", "-1/6", "-1/6"], ["-1/6", "1/6", "-1/6"],
       ["1/24", "1/12", "1/6"], ["1/24", "-1/12", "1/6"], [0, 0, 1]],
    AT=[[1, 1, 1, 1, 1, 0], [0, 1, -1, 2, -2, 0], [0, 1, 1, 4, 4, 0], [0, 1, -1, 8, -8, 1]],
    points="0,1,-1,2,-2,inf", m=4)


class _TS:
    def __init__(self, G, BT, AT, m):
        self.G = G
        self.BT = BT
        self.B = [list(r) for r in zip(*BT)]
        self.AT = AT
        self.A = [list(r) for r in zip(*AT)]
        self.n_o, self.n_h, self.mu = m, 3, len(G)
        self.n_x = m + 2


def _fr(M):
    return [[Fr(v) for v in r] for r in M]


@pytest.mark.parametrize("std", [LAVIN_F23, LAVIN_F43], ids=["F23", "F43"])
def test_toom_cook_reproduces_standard_matrices(std):
    G, BT, AT = _fr(std["G"]), _fr(std["BT"]), _fr(std["AT"])
    m = std["m"]
    # the standard matrices are an exact algorithm on their own
    std_ts = _TS(G, BT, AT, m)
    rng = random.Random(11)
    for _ in range(20):
        h = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(3)]
        x = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(m + 2)]
        assert CV.winograd_1d_exact(std_ts, h, x) == CV.direct_corr_1d(h, x)
    ts = T.make_transforms(std["points"], m)
    assert ts.mu == len(G)
    for i in range(ts.mu):
        # per point row: G_std = g_i G, BT_std = b_i BT, AT_std[:, i] = a_i AT[:, i]
        gi = _ratio(G[i], ts.G[i])
        bi = _ratio(BT[i], ts.BT[i])
        ai = _ratio([r[i] for r in AT], [r[i] for r in ts.AT])
        assert gi * bi * ai == 1


def _ratio(u, v):
    s = None
    for a, b in zip(u, v):
        if b == 0:
            assert a == 0
            continue
        r = Fr(a) / b
        assert s is None or s == r
        s = r
    assert s is not None and s != 0
    return s


def test_appendix_cfg3_matrices():
    """F(4,3) with points (0,-1,1,-1/2,1/2,inf): unscaled Vandermonde G."""
    ts = T.make_transforms("0,-1,1,-1/2,1/2,inf", 4)
    pts = [Fr(0), Fr(-1), Fr(1), Fr(-1, 2), Fr(1, 2)]
    assert ts.G[:5] == [[Fr(1), p, p * p] for p in pts]
    assert ts.G[5] == [0, 0, 1]
    assert ts.AT == [[p ** j for p in pts] + [Fr(0)] for j in range(3)] + \
        [[p ** 3 for p in pts] + [Fr(1)]]


# ------------------------------------------------------------------ counts


def _quads(k):
    qs = ["a^2+1", "a^2-2", "a^2+a+1", "a^2-a+1"]
    return [T.poly_mod(T.parse_poly(q)) for q in qs[:k]]


def _table1_config(n_o, lin, quad):
    use_inf = lin > 0
    nfin = lin - 1 if use_inf else lin
    mods = [T.point(p) for p in T.CANON_POINTS[:nfin]] + _quads(quad) + ([T.inf()] if use_inf else [])
    return mods


def test_table1():
    g = _gold("ratios.json")["table1"]
    for cell in g["cells"]:
        mods = _table1_config(cell["n_o"], cell["lin"], cell["quad"])
        assert T.validate(mods, cell["n_o"]) == [], cell
        ts = T.make_transforms(mods, cell["n_o"])
        r = T.ratio(mods, cell["n_o"])
        assert ts.mu ** 2 / Fr(cell["n_o"] ** 2) == r
        assert f"{float(r):.2f}".rstrip("0").rstrip(".") == cell["ratio"].rstrip("0").rstrip(".") or \
            abs(float(r) - float(cell["ratio"])) < 0.005, (cell, float(r))


def test_bullets_2x2():
    g = _gold("ratios.json")["bullets_2x2"]
    cfgs = [
        "0,-1,1,inf",                   # 4 linear (incl. inf)
        "0,a^2+1,inf",                  # 2 linear + 1 quadratic
        "a^3-2,inf",                    # 1 linear (inf) + 1 cubic
        "a^2+1,a^2-2",                  # 2 quadratics
        "a^4+1",                        # 1 quartic
    ]
    for spec, want in zip(cfgs, g["values"]):
        mods = T.parse_moduli(spec)
        assert T.validate(mods, 2) == [], spec
        ts = T.make_transforms(mods, 2)
        assert float(T.ratio(mods, 2)) == float(want)
        rng = random.Random(1)
        for _ in range(10):
            h = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(3)]
            x = [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(4)]
            assert CV.winograd_1d_exact(ts, h, x) == CV.direct_corr_1d(h, x), spec


def test_sec32_ratios():
    g = _gold("ratios.json")
    for n_o, want in zip(g["toom_cook_sec32"]["n_o"], g["toom_cook_sec32"]["values"]):
        mods = T.lin(n_o)
        assert round(float(T.ratio(mods, n_o)), 2) == float(want)
    for n_o, want in zip(g["winograd_a2p1_sec32"]["n_o"], g["winograd_a2p1_sec32"]["values"]):
        # linear points of TC(n_o - 2) plus one a^2 + 1
        # W(10), W(12) need 9 and 11 finite points; the printed list has 9, so
        # two further distinct points extend it (the count does not depend on them)
        pts = T.PAPER_POINTS + [Fr(1, 4), Fr(-4)]
        mods = [T.point(p) for p in pts[:n_o - 1]] + [T.poly_mod(T.parse_poly("a^2+1")), T.inf()]
        assert T.validate(mods, n_o) == []
        assert round(float(T.ratio(mods, n_o)), 2) == float(want)
    ex = g["example_ratios"]
    assert T.ratio(T.lin(2), 2) == Fr(ex["TC_2x2"])
    assert T.ratio(T.lin(4), 4) == Fr(ex["TC_4x4"])
    assert T.ratio(T.sup1(6), 6) == Fr(ex["W_6x6_one_quadratic"])


def test_optimal_toom_cook_count():
    """P:104 / P:498: all-linear (Toom-Cook) needs exactly mu = n_h + n_o - 1."""
    for m in range(2, 9):
        assert T.make_transforms(T.lin(m), m).mu == m + 2


# ------------------------------------------------------------------ brute-force exactness


def _rq(rng, n):
    return [Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(n)]


def _family():
    """SPEC acceptance 1: n_o in {2,4,6,8}; 0-2 quadratics from
    {a^2+1, a^2+a+1, a^2-a+1}; linear roots from the good-point list."""
    qs = ["a^2+1", "a^2+a+1", "a^2-a+1"]
    out = []
    for n_o in (2, 4, 6, 8):
        for nq in (0, 1, 2):
            for combo in itertools.combinations(qs, nq):
                nlin = n_o + 1 - 2 * nq
                if nlin < 0:
                    continue
                mods = [T.point(p) for p in T.PAPER_POINTS[:nlin]] + \
                    [T.poly_mod(T.parse_poly(q)) for q in combo] + [T.inf()]
                out.append((n_o, mods))
    return out


def test_exact_1d_family():
    rng = random.Random(2024)
    fam = _family()
    assert len(fam) >= 20
    for n_o, mods in fam:
        ts = T.make_transforms(mods, n_o)
        assert ts.mu == T.mu(mods)
        rb = T.residue_blocks(mods, n_o)
        for _ in range(25):
            h, x = _rq(rng, 3), _rq(rng, n_o + 2)
            ref = CV.direct_corr_1d(h, x)
            assert CV.winograd_1d_exact(ts, h, x) == ref, T.moduli_spec(mods)
            assert CV.residue_1d_exact(rb, h, x) == ref, T.moduli_spec(mods)


def test_exact_2d_tile_canonical_sets():
    rng = random.Random(99)
    for fam in ("lin", "sup1", "sup2"):
        for m in range(2, 9):
            if fam == "sup1" and m < 2 or fam == "sup2" and m < 2:
                continue
            mods, m = T.canonical(f"{fam}{m}")
            ts = T.make_transforms(mods, m)
            g = [_rq(rng, 3) for _ in range(3)]
            d = [_rq(rng, m + 2) for _ in range(m + 2)]
            ref = CV.direct_corr_2d(g, d)
            assert CV.winograd_2d_exact(ts, g, d) == ref, (fam, m)
            if m <= 6:
                rb = T.residue_blocks(mods, m)
                assert CV.residue_2d_exact(rb, g, d) == ref, (fam, m)


@pytest.mark.parametrize("name", ["lin2", "lin3", "sup1_2", "sup1_3", "sup2_4"])
def test_exact_tiled_layer_ragged(name):
    """Tiled multi-channel layer with pad 1 and ragged edges (5x7 image) equals
    direct convolution exactly (O8)."""
    rng = random.Random(len(name))
    mods, m = T.canonical(name)
    ts = T.make_transforms(mods, m)
    rb = T.residue_blocks(mods, m)
    x = [[[_rq(rng, 7) for _ in range(5)] for _ in range(2)]]
    w = [[[_rq(rng, 3) for _ in range(3)] for _ in range(2)] for _ in range(2)]
    for pad in (0, 1):
        ref = CV.direct_conv2d_exact(x, w, pad)
        assert CV.tiled_winograd_exact(ts, x, w, pad) == ref
        assert CV.tiled_residue_exact(rb, x, w, pad) == ref


def test_perturbed_matrix_fails():
    """a transform set with one entry perturbed by 1/1000 is not exact."""
    ts = T.make_transforms(T.lin(2), 2)
    ts.B[1][1] += Fr(1, 1000)
    rng = random.Random(3)
    h, x = _rq(rng, 3), _rq(rng, 4)
    assert CV.winograd_1d_exact(ts, h, x) != CV.direct_corr_1d(h, x)


def test_point_permutation_invariance():
    """permuting finite points permutes rows but not the result."""
    rng = random.Random(4)
    a = T.make_transforms("0,-1,1,-1/2,1/2,inf", 4)
    b = T.make_transforms("1/2,1,0,-1/2,-1,inf", 4)
    h, x = _rq(rng, 3), _rq(rng, 6)
    assert CV.winograd_1d_exact(a, h, x) == CV.winograd_1d_exact(b, h, x)


def test_residue_units():
    """(L + 4Q)^2 GEMM units for the residue lowering vs mu^2 = (L + 3Q)^2."""
    for name, L, Q in [("sup1_2", 2, 1), ("sup1_4", 4, 1), ("sup2_6", 4, 2), ("lin4", 6, 0)]:
        mods, m = T.canonical(name)
        rb = T.residue_blocks(mods, m)
        assert rb.units_1d == L + 4 * Q
        assert rb.D == m + 2 if any(x.is_inf for x in mods) else True
        assert T.mu(mods) == L + 3 * Q


# ------------------------------------------------------------------ validation


def test_validation_violations():
    v = T.validate(T.parse_moduli("0,a^2+a,inf"), 2)
    assert any("reducible" in s for s in v) and any("coprime" in s for s in v)
    v = T.validate(T.parse_moduli("1,1,-1,inf"), 2)
    assert any("coprime" in s for s in v)
    assert T.validate(T.parse_moduli("0,-1,inf"), 2)            # degree budget
    assert T.validate(T.parse_moduli("0,inf,-1,1"), 2)          # inf not last
    assert T.validate(T.parse_moduli("0,-1,1,inf"), 2) == []
    assert T.validate(T.parse_moduli("0,a^2+1,inf"), 2, sub_points=[Fr(0), Fr(0), T.INF])   # dup sub-points
    # sub-solver points may coincide with top-level points
    assert T.validate(T.parse_moduli("0,a^2+1,inf"), 2, sub_points=[Fr(0), Fr(-1), T.INF]) == []
    with pytest.raises(ValueError):
        T.make_transforms("0,-1,inf", 2)


def test_parse_moduli():
    mods = T.parse_moduli("0, -1, 1/2, a^2+1, a+1, inf")
    assert [str(m) for m in mods] == ["0", "-1", "1/2", "a^2+1", "-1", "inf"]
    assert T.parse_poly("a^2 - a + 1") == (Fr(1), Fr(-1), Fr(1))
    assert T.parse_poly("2*a^2-1/2") == (Fr(-1, 2), Fr(0), Fr(2))


@pytest.mark.parametrize("name", ["lin8", "lin6", "sup1_6", "sup2_6"])
def test_scaled_transforms_stay_exact(name):
    """Power-of-two point balancing (reading S1, [Vincent17] per P:607):
    the scaled algorithm still computes exact correlation (brute force on a
    random rational tile), the factors are powers of two, and for the
    Toom-Cook tiles the largest output weight shrinks (16384 -> 4 at m = 8)."""
    from fractions import Fraction
    import random
    mods, m = T.canonical(name)
    ts = T.make_transforms(mods, m)
    tss = T.scale_pow2_balance(ts)
    rnd = random.Random(3)
    g = [[Fraction(rnd.randint(-9, 9), rnd.randint(1, 4)) for _ in range(3)] for _ in range(3)]
    d = [[Fraction(rnd.randint(-9, 9), rnd.randint(1, 4)) for _ in range(m + 2)] for _ in range(m + 2)]
    assert CV.winograd_2d_exact(tss, g, d) == CV.direct_corr_2d(g, d)
    for i in range(ts.mu):
        ratios = {Fraction(tss.A[i][k]) / Fraction(ts.A[i][k]) for k in range(m) if ts.A[i][k] != 0}
        assert len(ratios) == 1
        f = ratios.pop()
        assert f.numerator & (f.numerator - 1) == 0 and f.denominator & (f.denominator - 1) == 0
    if name == "lin8":
        assert max(abs(a) for r in ts.A for a in r) == 16384
        assert max(abs(a) for r in tss.A for a in r) == 4


# Moduli of degree 3 and 4 ("1 polynomial of the first degree and 1 of
# the third degree", "1 polynomial of the fourth degree"; each degree-d modulus
# is solved by a Toom-Cook sub-problem on 2d - 1 points).
HIGHER_DEGREE = [("0,1,a^3+a+1,inf", 4), ("0,a^3-2,inf", 3), ("0,a^4+1,inf", 4), ("a^4+1,inf", 3),
                 ("a^3+2,a^2+1,inf", 4), ("a^3+a+1,inf", 2)]


@pytest.mark.parametrize("spec,m", HIGHER_DEGREE)
def test_exact_higher_degree_moduli(spec, m):
    """Generated transforms with cubic / quartic moduli compute the exact 1D and
    2D correlation (rational arithmetic vs brute force), in both lowerings, and
    the domain grows by 2d - 1 - d = d - 1 per degree-d modulus."""
    rng = random.Random(hash(spec) & 0xFFFF)
    mods = T.parse_moduli(spec)
    ts = T.make_transforms(mods, m)
    extra = sum(mm.degree - 1 for mm in mods if mm.degree and mm.degree > 1)
    assert ts.mu == m + 2 + extra
    rb = T.residue_blocks(mods, m)
    for _ in range(10):
        h, x = _rq(rng, 3), _rq(rng, m + 2)
        ref = CV.direct_corr_1d(h, x)
        assert CV.winograd_1d_exact(ts, h, x) == ref
        assert CV.residue_1d_exact(rb, h, x) == ref
    g = [_rq(rng, 3) for _ in range(3)]
    d = [_rq(rng, m + 2) for _ in range(m + 2)]
    assert CV.winograd_2d_exact(ts, g, d) == CV.direct_corr_2d(g, d)


@pytest.mark.parametrize("name", ["sup1_8", "sup1_10", "sup1_12", "sup2_12", "lin10"])
def test_exact_2d_tile_large_tiles(name):
    """Table 3's W(8x8) .. W(12x12) with one a^2+1, two
    quadratics at 12x12 and TC(10x10): exact 2D tile correlation in
    rational arithmetic; mu and the per-output ratio as Section 3.2 counts them."""
    rng = random.Random(len(name) * 7)
    mods, m = T.canonical(name)
    ts = T.make_transforms(mods, m)
    extra = 0 if name.startswith("lin") else int(name[3])   # sup1 / sup2: one / two quadratics
    assert ts.mu == m + 2 + extra
    if name.startswith("sup1"):
        assert abs(T.ratio(mods, m) - {8: 1.890625, 10: 1.69, 12: 225 / 144}[m]) < 1e-12   # Table 3 ratios
    g = [_rq(rng, 3) for _ in range(3)]
    d = [_rq(rng, m + 2) for _ in range(m + 2)]
    assert CV.winograd_2d_exact(ts, g, d) == CV.direct_corr_2d(g, d)
