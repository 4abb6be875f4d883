"""Pins for oracle/exact.py (O1): SPEC.md S:47-84 examples, randomized identities."""
import random
from fractions import Fraction as Fr

from oracle import exact as X


def P(*c):
    return X.norm([Fr(v) for v in c])


def test_mul_examples():
    assert X.mul(P(1, 1), P(1, -1)) == P(1, 0, -1)
    assert X.mul(P(3, 2, 1), P(1)) == P(3, 2, 1)
    assert X.mul(P(1, 2, 3), P(4, 5)) == P(4, 13, 22, 15)


def test_divmod_examples():
    assert X.divmod_(P(0, 0, 0, 1), P(1, 0, 1)) == (P(0, 1), P(0, -1))     # S:56 a^3 = a(a^2+1) - a
    assert X.divmod_(P(0, 0, 1), P(1, 1, 1)) == (P(1), P(-1, -1))
    assert X.divmod_(P(1, 2), P(0, 0, 1)) == ((), P(1, 2))


def test_gcd_examples():
    assert X.gcd(P(-1, 0, 1), P(-1, 1)) == P(-1, 1)
    assert X.gcd(P(0, 1), P(1, 0, 1)) == P(1)
    assert X.gcd(P(1, 1, 1), P(1, -1, 1)) == P(1)


def test_ext_euclid_examples():
    assert X.ext_euclid(P(0, 1), P(1, 0, 1)) == (P(1), P(0, -1))          # S:74, P:445 N_1 = 1
    assert X.ext_euclid(P(1, 0, 1), P(0, 1)) == (P(0, -1), P(1))          # S:75, P:445 N_2 = -a
    assert X.ext_euclid(P(-1, 1), P(0, 1)) == (P(1), P(-1))


def test_vec_examples():
    assert X.vec(P(1, 2, 3), 3) == [1, 2, 3]
    assert X.vec((), 2) == [0, 0]
    assert X.vec(P(1, 0, 1), 4) == [1, 0, 1, 0]


def _rand_poly(rng, d):
    return X.norm([Fr(rng.randint(-9, 9), rng.randint(1, 4)) for _ in range(d + 1)])


def test_random_identities():
    rng = random.Random(7)
    for _ in range(300):
        p = _rand_poly(rng, rng.randint(0, 6))
        m = _rand_poly(rng, rng.randint(1, 4))
        if not m or X.deg(m) < 1:
            continue
        q, r = X.divmod_(p, m)
        assert X.add(X.mul(q, m), r) == p
        assert X.deg(r) < X.deg(m)
        M = _rand_poly(rng, rng.randint(1, 4))
        if X.deg(M) < 1 or X.deg(X.gcd(m, M)) > 0:
            continue
        N, n = X.ext_euclid(m, M)
        assert X.add(X.mul(N, M), X.mul(n, m)) == (Fr(1),)
        assert X.deg(N) < X.deg(m)


def test_field_axioms():
    rng = random.Random(3)
    for _ in range(200):
        a, b, c = (_rand_poly(rng, rng.randint(0, 3)) for _ in range(3))
        assert X.mul(a, X.add(b, c)) == X.add(X.mul(a, b), X.mul(a, c))
        assert X.mul(X.mul(a, b), c) == X.mul(a, X.mul(b, c))
        assert X.sub(X.add(a, b), b) == a


def test_reducibility():
    assert not X.has_rational_root(P(1, 0, 1))      # a^2 + 1
    assert not X.has_rational_root(P(-2, 0, 1))     # a^2 - 2
    assert not X.has_rational_root(P(1, 1, 1))      # a^2 + a + 1
    assert X.has_rational_root(P(0, 1, 1))          # a^2 + a = a (a + 1)
    assert X.has_rational_root(P(Fr(-1, 4), 0, 1))  # (a - 1/2)(a + 1/2)
