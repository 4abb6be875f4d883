"""Transform generation (oracle components O2-O6).  Test infrastructure only.

Follows PAPER.md Sec. 2.2 step by step:

* O2  Toom-Cook sub-solver F_TC(d x d, d x d) in the paper's convention
      (P:242-243): G^(TC) rows carry N_i = 1/M_i(q_i),
      A^(TC) rows are plain evaluations, B^(TC) column i = vec(M_i(a)), the
      pseudo-point column = vec(M(a)).
* O3  Algorithm 1: G^W, A^W.  Linear moduli -> unscaled Vandermonde
      rows ("not scaled by factors N_i"); degree-d moduli -> G^(TC) G' and
      A^(TC) A'; pseudo-point infinity -> [0 ... 0 1].
      Reading A1: A' has n_o columns j = 0..n_o-1 as Algorithm 1
      states; the 4-column A' of the worked example is an erratum.
* O4  Algorithm 2: C = blockdiag(C_i), E_i = vec(R_M[a^k N_i M_i]),
      zero row appended to E iff infinity is used, B^W = [E C | vec M].
      Reading A2: N_i comes from the extended Euclidean algorithm; the
      printed N_1 = 1, N_2 = -a hold only for b = 0, c = 1.
* O5  Role assignment for the correlation form of Eq. (2):
      y = A^T [(G g) (.) (B^T d)] with G := G^W (mu x n_h), B := B^W (n_x x mu),
      A := A^W (mu x n_o).  Reading A4.
* O6  Residue-block matrices for the "any suitable algorithm" sub-problem solver
      of P:107: the degree-d residue product mod m_i is computed directly as a
      d x d block (multiplication by a^k mod m_i), instead of by F_TC.
"""
from dataclasses import dataclass
from fractions import Fraction
import re

from . import exact as X

INF = "inf"

# "known good root points: 0, -1, 1, -1/2, 2, 1/2, -2, -1/4, 4".
PAPER_POINTS = [Fraction(0), Fraction(-1), Fraction(1), Fraction(-1, 2), Fraction(2),
                Fraction(1, 2), Fraction(-2), Fraction(-1, 4), Fraction(4)]
# the same points reordered so the first five are BASELINE cfg3's set,
# then 1/4, -4 (reading A21: P:533 lists nine points, Table 3's W(12x12)
# takes TC(10x10)'s eleven; the list continues its +-2^k alternation).
CANON_POINTS = [Fraction(0), Fraction(-1), Fraction(1), Fraction(-1, 2), Fraction(1, 2),
                Fraction(2), Fraction(-2), Fraction(-1, 4), Fraction(4), Fraction(1, 4), Fraction(-4)]
# "To solve the subproblem ... we use F_TC(2x2, 2x2) and root points 0, -1 and inf".
DEFAULT_SUB_POINTS = [Fraction(0), Fraction(-1), INF]


@dataclass(frozen=True)
class Modulus:
    """One CRT modulus m_i(a): a monic polynomial of degree >= 1, or the
    pseudo-point infinity."""
    poly: tuple  # monic, constant first; () for infinity

    @property
    def is_inf(self):
        return self.poly == ()

    @property
    def degree(self):
        return 0 if self.is_inf else len(self.poly) - 1

    @property
    def root(self):
        assert self.degree == 1
        return -self.poly[0]

    def __str__(self):
        if self.is_inf:
            return "inf"
        if self.degree == 1:
            return str(self.root)
        return poly_str(self.poly)


def poly_str(p):
    terms = []
    for k in range(len(p) - 1, -1, -1):
        c = p[k]
        if c == 0:
            continue
        mono = "" if k == 0 else ("a" if k == 1 else f"a^{k}")
        if mono and abs(c) == 1:
            s = mono
        else:
            s = f"{abs(c)}" + (f"*{mono}" if mono else "")
        terms.append(("-" if c < 0 else "+") + s)
    out = "".join(terms)
    return out[1:] if out.startswith("+") else out


def point(p):
    return Modulus(X.linear(p))


def inf():
    return Modulus(())


def poly_mod(coeffs):
    return Modulus(X.monic(coeffs))


_TERM = re.compile(r"([+-]?)\s*([0-9/]*)\s*\*?\s*(a(?:\^([0-9]+))?)?")


def parse_poly(s):
    """Parse 'a^2+a+1', 'a^2-2', 'a+1', '2*a^2-1' into a coefficient tuple."""
    s = s.replace(" ", "").replace("**", "^")
    if not s:
        raise ValueError("empty polynomial")
    coeffs = {}
    pos = 0
    while pos < len(s):
        m = _TERM.match(s, pos)
        if not m or m.end() == pos:
            raise ValueError(f"cannot parse polynomial {s!r}")
        sign, num, mono, power = m.groups()
        if not num and not mono:
            raise ValueError(f"cannot parse polynomial {s!r}")
        c = Fraction(num) if num else Fraction(1)
        if sign == "-":
            c = -c
        k = 0 if not mono else (int(power) if power else 1)
        coeffs[k] = coeffs.get(k, Fraction(0)) + c
        pos = m.end()
    n = max(coeffs) + 1
    return X.norm([coeffs.get(i, Fraction(0)) for i in range(n)])


def parse_moduli(spec):
    """'0,-1,1/2,a^2+1,inf' -> [Modulus].  A bare rational p is the point p
    (modulus a - p); a token containing 'a' is a polynomial modulus (degree-1
    polynomials become points); 'inf' is the pseudo-point."""
    out = []
    for tok in spec.split(","):
        tok = tok.strip()
        if tok.lower() in ("inf", "infinity", "∞"):
            out.append(inf())
        elif "a" in tok:
            out.append(poly_mod(parse_poly(tok)))
        else:
            out.append(point(Fraction(tok)))
    return out


def parse_points(spec):
    out = []
    for tok in spec.split(","):
        tok = tok.strip()
        out.append(INF if tok.lower() in ("inf", "infinity", "∞") else Fraction(tok))
    return out


# --------------------------------------------------------------------------- O2


def toom_cook_subsolver(points, d):
    """F_TC(d x d, d x d) in the paper's convention.

    Returns (G_tc, A_tc, B_tc) with shapes (2d-1) x d, (2d-1) x d,
    (2d-1) x (2d-1) such that, for polynomials u, x with d coefficients,
    vec(u*x) = B_tc [(G_tc u) (.) (A_tc x)].  Row / column order follows the
    point order; infinity (if present) must be last.
    """
    if len(points) != 2 * d - 1:
        raise ValueError(f"sub-solver for degree {d} needs {2 * d - 1} points")
    finite = [p for p in points if p != INF]
    if len(set(finite)) != len(finite) or points.count(INF) > 1:
        raise ValueError("sub-solver points must be distinct")
    if INF in points and points[-1] != INF:
        raise ValueError("the pseudo-point inf must be the last sub-solver point")
    n = 2 * d - 1
    Msub = X.prod([X.linear(q) for q in finite])
    G, A, Bcols = [], [], []
    for q in points:
        if q == INF:
            G.append([Fraction(0)] * (d - 1) + [Fraction(1)])
            A.append([Fraction(0)] * (d - 1) + [Fraction(1)])
            Bcols.append(X.vec(Msub, n))
        else:
            Mi = X.divmod_(Msub, X.linear(q))[0]
            Ni = 1 / X.evaluate(Mi, q)
            G.append([Ni * q ** j for j in range(d)])
            A.append([q ** j for j in range(d)])
            Bcols.append(X.vec(Mi, n))
    B = [[Bcols[j][i] for j in range(n)] for i in range(n)]
    return G, A, B


def default_sub_points(d):
    """2d-1 sub-solver points: the first 2d-2 paper points plus infinity.  For
    d = 2 this is {0, -1, inf} exactly as P:533 states."""
    return PAPER_POINTS[:2 * d - 2] + [INF]


# --------------------------------------------------------------------------- validation


def validate(moduli, n_o, n_h=3, sub_points=None):
    """List of violations (empty iff the configuration is valid).

    P:83 / P:319 / P:376: irreducible, pairwise coprime moduli with
    sum deg = n_h + n_o - 2 when the pseudo-point is used, and
    n_h + n_o - 1 without it (reading A7).  P:108: coprimality is required
    only within a level, so sub-solver points may repeat top-level points.
    """
    v = []
    n_inf = sum(1 for m in moduli if m.is_inf)
    if n_inf > 1:
        v.append("pseudo-point inf appears more than once")
    if n_inf == 1 and not moduli[-1].is_inf:
        v.append("pseudo-point inf must be the last modulus")
    finite = [m for m in moduli if not m.is_inf]
    need = n_h + n_o - 2 if n_inf else n_h + n_o - 1
    have = sum(m.degree for m in finite)
    if have != need:
        v.append(f"degree budget: sum deg = {have}, need {need} (n_o={n_o}, n_h={n_h}, inf={bool(n_inf)})")
    for i, m in enumerate(finite):
        if m.degree == 2 and X.has_rational_root(m.poly):
            v.append(f"modulus {m} is reducible over Q")
        for mm in finite[i + 1:]:
            if X.deg(X.gcd(m.poly, mm.poly)) > 0:
                v.append(f"moduli {m} and {mm} are not coprime")
    for m in finite:
        if m.degree >= 2:
            sp = sub_points_for(m, sub_points)
            if len(sp) != 2 * m.degree - 1:
                v.append(f"modulus {m}: sub-solver needs {2 * m.degree - 1} points, got {len(sp)}")
            fin = [p for p in sp if p != INF]
            if len(set(fin)) != len(fin) or sp.count(INF) > 1:
                v.append(f"modulus {m}: duplicate sub-solver points")
            elif INF in sp and sp[-1] != INF:
                v.append(f"modulus {m}: inf must be the last sub-solver point")
    return v


def sub_points_for(m, sub_points):
    if sub_points is None:
        return default_sub_points(m.degree)
    if isinstance(sub_points, dict):
        return sub_points.get(m.degree, default_sub_points(m.degree))
    return list(sub_points)


def mu(moduli):
    """Winograd-domain size per dimension (Sec. 2.3): every degree-d
    modulus solved by F_TC(d x d, d x d) costs 2d - 1 points (linear: 1), the
    pseudo-point costs 1.  Reading A7."""
    return sum(1 if m.is_inf else 2 * m.degree - 1 for m in moduli)


def ratio(moduli, n_o, dims=2):
    """Multiplications per output point: mu^2 / n_o^2 in 2D, mu / n_o in 1D."""
    u = mu(moduli)
    return Fraction(u ** dims, n_o ** dims)


# --------------------------------------------------------------------------- O3 / O4


def algorithm1(moduli, n_o, n_h=3, sub_points=None):
    """Algorithm 1: returns (G^W, A^W) as lists of rows."""
    G, A = [], []
    for m in moduli:
        if m.is_inf:
            continue
        d = m.degree
        if d == 1:
            p = m.root
            G.append([p ** j for j in range(n_h)])
            A.append([p ** j for j in range(n_o)])
        else:
            Gp = _residue_map(m.poly, n_h)   # d x n_h, columns vec(R_m[a^j])
            Ap = _residue_map(m.poly, n_o)   # d x n_o  (reading A1)
            Gtc, Atc, _ = toom_cook_subsolver(sub_points_for(m, sub_points), d)
            G.extend(_matmul(Gtc, Gp))
            A.extend(_matmul(Atc, Ap))
    if any(m.is_inf for m in moduli):
        G.append([Fraction(0)] * (n_h - 1) + [Fraction(1)])
        A.append([Fraction(0)] * (n_o - 1) + [Fraction(1)])
    return G, A


def algorithm2(moduli, n_o, n_h=3, sub_points=None, return_parts=False):
    """Algorithm 2: B^W = [E C | vec M] (no vec M column and no
    appended zero row of E without the pseudo-point)."""
    finite = [m for m in moduli if not m.is_inf]
    has_inf = len(finite) != len(moduli)
    Mpoly = X.prod([m.poly for m in finite])
    degM = X.deg(Mpoly)
    # C = blockdiag(C_i)
    blocks = []
    for m in finite:
        d = m.degree
        if d == 1:
            blocks.append([[Fraction(1)]])
        else:
            _, _, Btc = toom_cook_subsolver(sub_points_for(m, sub_points), d)
            ncol = 2 * d - 1
            cols = []
            for j in range(ncol):
                bj = X.norm([Btc[i][j] for i in range(ncol)])     # b_j(a)
                cols.append(X.vec(X.rem(bj, m.poly), d))
            blocks.append([[cols[j][i] for j in range(ncol)] for i in range(d)])
    C = _blockdiag(blocks)
    # E = [E_1 ... E_l] (+ zero row)
    Ecols = []
    for m in finite:
        Mi = X.divmod_(Mpoly, m.poly)[0]
        Ni, _ = X.ext_euclid(m.poly, Mi)
        for k in range(m.degree):
            Ecols.append(X.vec(X.rem(X.mul(X.monomial(k), X.mul(Ni, Mi)), Mpoly), degM))
    E = [[Ecols[j][i] for j in range(len(Ecols))] for i in range(degM)]
    if has_inf:
        E.append([Fraction(0)] * len(Ecols))
    EC = _matmul(E, C)
    if has_inf:
        vm = X.vec(Mpoly, degM + 1)
        B = [row + [vm[i]] for i, row in enumerate(EC)]
    else:
        B = EC
    if return_parts:
        return B, C, E
    return B


@dataclass
class TransformSet:
    """Exact matrices of one algorithm in the correlation role assignment (O5):
    y = A^T [(G g) (.) (B^T d)];  G: mu x n_h, B: n_x x mu, A: mu x n_o."""
    moduli: list
    n_o: int
    n_h: int
    G: list
    B: list
    A: list

    @property
    def mu(self):
        return len(self.G)

    @property
    def n_x(self):
        return self.n_o + self.n_h - 1

    @property
    def BT(self):
        return _transpose(self.B)

    @property
    def AT(self):
        return _transpose(self.A)


def make_transforms(moduli, n_o, n_h=3, sub_points=None):
    if isinstance(moduli, str):
        moduli = parse_moduli(moduli)
    v = validate(moduli, n_o, n_h, sub_points)
    if v:
        raise ValueError("; ".join(v))
    G, A = algorithm1(moduli, n_o, n_h, sub_points)
    B = algorithm2(moduli, n_o, n_h, sub_points)
    ts = TransformSet(list(moduli), n_o, n_h, G, B, A)
    assert len(G) == mu(moduli) == len(A) == len(B[0]), "mu consistency"
    assert len(B) == n_o + n_h - 1
    return ts


# --------------------------------------------------------------------------- scaled transforms


def _pow2_floor_log2(r):
    """e with 2^e <= r < 2^(e+1) for a positive Fraction r (exact)."""
    r = Fraction(r)
    e = r.numerator.bit_length() - r.denominator.bit_length()
    while Fraction(2) ** e > r:
        e -= 1
    while Fraction(2) ** (e + 1) <= r:
        e += 1
    return e


def scale_pow2_balance(ts):
    """Power-of-two diagonal rescaling of the Winograd points (the "scaled G and
    A^T" conditioning trick of [Vincent17] that P:607 lists as composable with
    the method; reading S1).  Point i's input-transform row (column i
    of B) is multiplied by 2^-s_i and its output-transform row (row i of A) by
    2^s_i, with s_i = floor(floor(log2(max|B[:, i]| / max|A[i, :]|)) / 2), so the
    two magnitudes meet halfway.  The product A^T[(G g) (.) (B^T d)] is unchanged
    exactly (each Hadamard term gains 2^-s_i and loses it again), and powers of
    two are exact in every floating-point format."""
    mu = ts.mu
    B = [list(r) for r in ts.B]
    A = [list(r) for r in ts.A]
    for i in range(mu):
        bmax = max(abs(Fraction(B[j][i])) for j in range(len(B)))
        amax = max(abs(Fraction(a)) for a in A[i])
        if bmax == 0 or amax == 0:
            continue
        s = _pow2_floor_log2(bmax / amax) // 2
        f = Fraction(2) ** s
        for j in range(len(B)):
            B[j][i] = Fraction(B[j][i]) / f
        A[i] = [Fraction(a) * f for a in A[i]]
    return TransformSet(list(ts.moduli), ts.n_o, ts.n_h, [list(r) for r in ts.G], B, A)


# --------------------------------------------------------------------------- O6


@dataclass
class ResidueBlocks:
    """Residue-block lowering (O6).  Per dimension D = sum of block sizes
    coordinates (linear / infinity: 1; degree d: d residue coefficients).

    1D correlation:  y = A_P^T  blockdiag_i( Phi(u_i)^T ) B_P^T d,  u = G_P g,
    with Phi(u_i) = sum_k u_{i,k} Phi_{i,k} and Phi_{i,k} the d x d matrix of
    multiplication by a^k modulo m_i (column j = vec(R_{m_i}[a^{k+j}])).
    """
    moduli: list
    n_o: int
    n_h: int
    GP: list       # D x n_h
    BP: list       # n_x x D   (E_full = [E | vec M])
    AP: list       # D x n_o
    blocks: list   # [(start, size, Modulus)]
    phi: list      # per block: list of size x size matrices Phi_k, k < size

    @property
    def D(self):
        return len(self.GP)

    @property
    def units_1d(self):
        return sum(s * s for _, s, _ in self.blocks)


def residue_blocks(moduli, n_o, n_h=3):
    if isinstance(moduli, str):
        moduli = parse_moduli(moduli)
    v = validate(moduli, n_o, n_h, None)
    if v:
        raise ValueError("; ".join(v))
    finite = [m for m in moduli if not m.is_inf]
    has_inf = len(finite) != len(moduli)
    GP, AP, blocks, phi = [], [], [], []
    for m in finite:
        d = m.degree
        start = len(GP)
        Gp = _residue_map(m.poly, n_h)
        Ap = _residue_map(m.poly, n_o)
        GP.extend(Gp)
        AP.extend(Ap)
        blocks.append((start, d, m))
        phi.append([_mult_matrix(m.poly, k) for k in range(d)])
    if has_inf:
        blocks.append((len(GP), 1, inf()))
        GP.append([Fraction(0)] * (n_h - 1) + [Fraction(1)])
        AP.append([Fraction(0)] * (n_o - 1) + [Fraction(1)])
        phi.append([[[Fraction(1)]]])
    _, _, E = algorithm2(moduli, n_o, n_h, None, return_parts=True)
    if has_inf:
        Mpoly = X.prod([m.poly for m in finite])
        vm = X.vec(Mpoly, X.deg(Mpoly) + 1)
        BP = [row + [vm[i]] for i, row in enumerate(E)]
    else:
        BP = [list(r) for r in E]
    return ResidueBlocks(list(moduli), n_o, n_h, GP, BP, AP, blocks, phi)


def residue_weight_1d(rb, u):
    """W[(k),(k')] such that z = W v  for one 1D tile: block i contributes
    Phi(u_i)^T.  Returns a D x D matrix (block diagonal)."""
    D = rb.D
    W = [[Fraction(0)] * D for _ in range(D)]
    for (start, size, _), phis in zip(rb.blocks, rb.phi):
        for k in range(size):
            for r in range(size):
                for c in range(size):
                    W[start + r][start + c] += u[start + k] * phis[k][c][r]   # Phi^T
    return W


# --------------------------------------------------------------------------- helpers


def _residue_map(mpoly, ncols):
    """d x ncols matrix whose column j is vec(R_m[a^j])."""
    d = X.deg(mpoly)
    cols = [X.vec(X.rem(X.monomial(j), mpoly), d) for j in range(ncols)]
    return [[cols[j][i] for j in range(ncols)] for i in range(d)]


def _mult_matrix(mpoly, k):
    """Matrix of v(a) -> R_m[a^k v(a)] on vec coordinates (column j = vec(R_m[a^{k+j}]))."""
    d = X.deg(mpoly)
    cols = [X.vec(X.rem(X.monomial(k + j), mpoly), d) for j in range(d)]
    return [[cols[j][i] for j in range(d)] for i in range(d)]


def _matmul(P, Q):
    n, k, m = len(P), len(Q), len(Q[0])
    assert all(len(r) == k for r in P)
    return [[sum((P[i][t] * Q[t][j] for t in range(k)), Fraction(0)) for j in range(m)] for i in range(n)]


def _transpose(P):
    return [list(r) for r in zip(*P)]


def _blockdiag(blocks):
    R = sum(len(b) for b in blocks)
    Cn = sum(len(b[0]) for b in blocks)
    out = [[Fraction(0)] * Cn for _ in range(R)]
    r0 = c0 = 0
    for b in blocks:
        for i, row in enumerate(b):
            for j, v in enumerate(row):
                out[r0 + i][c0 + j] = v
        r0 += len(b)
        c0 += len(b[0])
    return out


# --------------------------------------------------------------------------- canonical sets


def lin(m):
    """lin(m) = P[:m+1] + {inf}, mu = m + 2 (canonical sets)."""
    return [point(p) for p in CANON_POINTS[:m + 1]] + [inf()]


def sup1(m):
    """sup1(m) = P[:m-1] + {a^2+1, inf}, mu = m + 3."""
    return [point(p) for p in CANON_POINTS[:m - 1]] + [poly_mod(parse_poly("a^2+1")), inf()]


def sup2(m):
    """sup2(m) = P[:m-3] + {a^2+1, a^2-2, inf}; at m = 2: {a^2+1, a^2-2}, no inf."""
    q = [poly_mod(parse_poly("a^2+1")), poly_mod(parse_poly("a^2-2"))]
    if m == 2:
        return q
    return [point(p) for p in CANON_POINTS[:m - 3]] + q + [inf()]


def canonical(name):
    """'lin4', 'sup1_6', 'sup2_8' -> moduli list, m."""
    mt = re.fullmatch(r"(lin|sup1|sup2)_?(\d+)", name)
    if not mt:
        raise ValueError(name)
    fam, m = mt.group(1), int(mt.group(2))
    return {"lin": lin, "sup1": sup1, "sup2": sup2}[fam](m), m


def moduli_spec(moduli):
    return ",".join(str(m) for m in moduli)
