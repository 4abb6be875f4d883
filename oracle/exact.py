"""Exact polynomial algebra over Q (oracle component O1).

PAPER.md P:83-88 (CRT over F[a], Eq. 1), P:90-91 (residues mod m_i),
P:240-241 (vec(.) and R_m[.]), P:406 (extended Euclidean algorithm).

A polynomial is a tuple of ``fractions.Fraction`` with the constant term first
(vec(m(a)) = [m_1 ... m_n]^T for m(a) = m_1 + m_2 a + ... ).  The zero
polynomial is the empty tuple.  Test infrastructure only (see oracle/__init__).
"""
import math
from fractions import Fraction

Poly = tuple


def F(v):
    """Coerce an int / str / Fraction to Fraction."""
    return v if isinstance(v, Fraction) else Fraction(v)


def norm(p):
    """Strip trailing (leading-degree) zeros so deg = len - 1."""
    p = [F(c) for c in p]
    while p and p[-1] == 0:
        p.pop()
    return tuple(p)


def deg(p):
    p = norm(p)
    return len(p) - 1 if p else -1


def add(p, q):
    n = max(len(p), len(q))
    return norm([(p[i] if i < len(p) else 0) + (q[i] if i < len(q) else 0) for i in range(n)])


def neg(p):
    return tuple(-c for c in norm(p))


def sub(p, q):
    return add(p, neg(q))


def scale(p, s):
    return norm([F(s) * c for c in p])


def mul(p, q):
    """Polynomial product: coefficients are the linear convolution of the
    coefficient vectors ('convolution can be expressed as polynomial
    multiplication')."""
    p, q = norm(p), norm(q)
    if not p or not q:
        return ()
    out = [Fraction(0)] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        for j, b in enumerate(q):
            out[i + j] += a * b
    return norm(out)


def divmod_(p, m):
    """(quotient, remainder) with p = q*m + r, deg r < deg m.  The remainder is
    the paper's R_{m(a)}[p(a)]."""
    p, m = list(norm(p)), norm(m)
    if not m:
        raise ZeroDivisionError("division by the zero polynomial")
    dm = len(m) - 1
    lead = m[-1]
    q = [Fraction(0)] * max(len(p) - dm, 1)
    while len(p) - 1 >= dm and p:
        k = len(p) - 1 - dm
        c = p[-1] / lead
        q[k] = c
        for i, mc in enumerate(m):
            p[i + k] -= c * mc
        p = list(norm(p))
    return norm(q), norm(p)


def rem(p, m):
    """R_{m(a)}[p(a)]."""
    return divmod_(p, m)[1]


def monic(p):
    p = norm(p)
    return scale(p, 1 / p[-1]) if p else ()


def gcd(p, q):
    """Monic greatest common divisor (Euclid)."""
    p, q = norm(p), norm(q)
    if not p and not q:
        raise ValueError("gcd(0, 0) undefined")
    while q:
        p, q = q, rem(p, q)
    return monic(p)


def ext_euclid(m, M):
    """Return (N, n) with N*M + n*m = 1, deg N < deg m ('N_i(a) --
    polynomial obtained from extended Euclidean algorithm for m_i(a) and
    M_i(a)').  Raises ValueError when gcd(m, M) != 1."""
    m, M = norm(m), norm(M)
    # invariant: r_i = s_i*M + t_i*m
    r0, s0, t0 = M, (Fraction(1),), ()
    r1, s1, t1 = m, (), (Fraction(1),)
    while r1:
        qt, r2 = divmod_(r0, r1)
        s2 = sub(s0, mul(qt, s1))
        t2 = sub(t0, mul(qt, t1))
        r0, s0, t0, r1, s1, t1 = r1, s1, t1, r2, s2, t2
    if deg(r0) != 0:
        raise ValueError("ext_euclid: inputs are not coprime")
    c = r0[0]
    N, n = scale(s0, 1 / c), scale(t0, 1 / c)
    # reduce N modulo m so deg N < deg m (adjust n accordingly)
    if deg(m) > 0 and deg(N) >= deg(m):
        qt, N = divmod_(N, m)
        n = add(n, mul(qt, M))
    assert add(mul(N, M), mul(n, m)) == (Fraction(1),)
    return N, n


def vec(p, length):
    """vec(p(a)) zero-padded to ``length`` entries, constant first."""
    p = norm(p)
    if len(p) > length:
        raise ValueError("vec: polynomial longer than requested length")
    return [p[i] if i < len(p) else Fraction(0) for i in range(length)]


def evaluate(p, x):
    x = F(x)
    acc = Fraction(0)
    for c in reversed(norm(p)):
        acc = acc * x + c
    return acc


def prod(polys):
    out = (Fraction(1),)
    for p in polys:
        out = mul(out, p)
    return out


def monomial(k):
    """a^k."""
    return tuple([Fraction(0)] * k + [Fraction(1)])


def linear(p):
    """The linear modulus a - p (a 'point' p)."""
    return (-F(p), Fraction(1))


def has_rational_root(p):
    """True iff the degree-2 polynomial p has a rational root (reducible over Q).
    Used for the irreducibility requirement of P:83 / P:319 (degree 2 only)."""
    p = monic(p)
    if deg(p) != 2:
        raise ValueError("has_rational_root: degree-2 polynomials only")
    c, b = p[0], p[1]
    disc = b * b - 4 * c
    if disc < 0:
        return False
    num, den = disc.numerator, disc.denominator
    rn, rd = math.isqrt(num), math.isqrt(den)
    return rn * rn == num and rd * rd == den
