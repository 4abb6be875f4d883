// exact.hpp -- overflow-checked exact rationals and polynomials over Q for the
// host-side CRT transform generator (Sec. 2.1: "ring of polynomials
// over a field F", Eq. 1; P:240-241 vec(.) and R_m[.]).  Entries of every
// transform this library generates stay far inside 64 bits (m <= 8); any
// intermediate that would leave __int128 raises RangeError -> WINO_E_RANGE.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace wino {

struct RangeError : std::runtime_error {
  explicit RangeError(const std::string& s) : std::runtime_error(s) {}
};
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& s) : std::runtime_error(s) {}
};

using i128 = __int128;

inline i128 iabs(i128 a) { return a < 0 ? -a : a; }
inline i128 igcd(i128 a, i128 b) {
  a = iabs(a);
  b = iabs(b);
  while (b) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
inline i128 mul_ck(i128 a, i128 b) {
  i128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw RangeError("rational overflow (mul)");
  return r;
}
inline i128 add_ck(i128 a, i128 b) {
  i128 r;
  if (__builtin_add_overflow(a, b, &r)) throw RangeError("rational overflow (add)");
  return r;
}

// Reduced rational n/d with d > 0.
struct Rat {
  i128 n = 0, d = 1;
  Rat() = default;
  Rat(long long v) : n(v), d(1) {}  // NOLINT: implicit from integer literals
  static Rat make(i128 n, i128 d) {
    if (d == 0) throw std::domain_error("division by zero");
    if (d < 0) n = -n, d = -d;
    i128 g = igcd(n, d);
    if (g > 1) n /= g, d /= g;
    Rat r;
    r.n = n;
    r.d = d;
    return r;
  }
  bool is_zero() const { return n == 0; }
};

inline Rat operator+(const Rat& a, const Rat& b) {
  i128 g = igcd(a.d, b.d);
  i128 da = a.d / g, db = b.d / g;
  return Rat::make(add_ck(mul_ck(a.n, db), mul_ck(b.n, da)), mul_ck(a.d, db));
}
inline Rat operator-(const Rat& a) { return Rat::make(-a.n, a.d); }
inline Rat operator-(const Rat& a, const Rat& b) { return a + (-b); }
inline Rat operator*(const Rat& a, const Rat& b) {
  i128 g1 = igcd(a.n, b.d), g2 = igcd(b.n, a.d);
  if (g1 == 0) g1 = 1;
  if (g2 == 0) g2 = 1;
  return Rat::make(mul_ck(a.n / g1, b.n / g2), mul_ck(a.d / g2, b.d / g1));
}
inline Rat operator/(const Rat& a, const Rat& b) {
  if (b.n == 0) throw std::domain_error("division by zero rational");
  return a * Rat::make(b.d, b.n);
}
inline bool operator==(const Rat& a, const Rat& b) { return a.n == b.n && a.d == b.d; }
inline bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
inline bool operator<(const Rat& a, const Rat& b) { return mul_ck(a.n, b.d) < mul_ck(b.n, a.d); }

// Polynomial, constant term first, normalised: no trailing zeros.
using Poly = std::vector<Rat>;

inline void pnorm(Poly& p) {
  while (!p.empty() && p.back().is_zero()) p.pop_back();
}
inline int pdeg(const Poly& p) { return static_cast<int>(p.size()) - 1; }  // zero poly -> -1

inline Poly padd(const Poly& a, const Poly& b) {
  Poly r(std::max(a.size(), b.size()));
  for (size_t i = 0; i < r.size(); ++i) r[i] = (i < a.size() ? a[i] : Rat()) + (i < b.size() ? b[i] : Rat());
  pnorm(r);
  return r;
}
inline Poly pscale(const Poly& a, const Rat& s) {
  Poly r(a.size());
  for (size_t i = 0; i < a.size(); ++i) r[i] = a[i] * s;
  pnorm(r);
  return r;
}
inline Poly psub(const Poly& a, const Poly& b) { return padd(a, pscale(b, Rat(-1))); }
inline Poly pmul(const Poly& a, const Poly& b) {
  if (a.empty() || b.empty()) return {};
  Poly r(a.size() + b.size() - 1);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) r[i + j] = r[i + j] + a[i] * b[j];
  pnorm(r);
  return r;
}
// Long division: a = q*b + r, deg r < deg b.  r is R_b[a].
inline void pdivmod(const Poly& a, const Poly& b, Poly& q, Poly& r) {
  if (b.empty()) throw std::domain_error("polynomial division by zero");
  r = a;
  pnorm(r);
  int db = pdeg(b);
  q.assign(std::max<int>(pdeg(r) - db + 1, 0), Rat());
  while (!r.empty() && pdeg(r) >= db) {
    int k = pdeg(r) - db;
    Rat c = r.back() / b.back();
    q[k] = c;
    for (int i = 0; i <= db; ++i) r[i + k] = r[i + k] - c * b[i];
    pnorm(r);
  }
  pnorm(q);
}
inline Poly prem(const Poly& a, const Poly& b) {
  Poly q, r;
  pdivmod(a, b, q, r);
  return r;
}
inline Poly pquo(const Poly& a, const Poly& b) {
  Poly q, r;
  pdivmod(a, b, q, r);
  return q;
}
inline Poly pmonomial(int k) {
  Poly p(k + 1);
  p[k] = Rat(1);
  return p;
}
inline Poly plinear(const Rat& root) { return Poly{-root, Rat(1)}; }  // a - p
inline Rat peval(const Poly& p, const Rat& x) {
  Rat acc;
  for (int i = pdeg(p); i >= 0; --i) acc = acc * x + p[i];
  return acc;
}
inline Poly pmonic(const Poly& p) { return p.empty() ? p : pscale(p, Rat(1) / p.back()); }
inline Poly pgcd(Poly a, Poly b) {
  pnorm(a);
  pnorm(b);
  while (!b.empty()) {
    Poly r = prem(a, b);
    a = b;
    b = r;
  }
  return pmonic(a);
}
// vec(p) zero-padded to `len`.
inline std::vector<Rat> pvec(const Poly& p, int len) {
  if (pdeg(p) >= len) throw std::logic_error("vec: polynomial too long");
  std::vector<Rat> v(len);
  for (size_t i = 0; i < p.size(); ++i) v[i] = p[i];
  return v;
}
// Extended Euclid: N*M + n*m = 1 with deg N < deg m.  Returns N.
inline Poly ext_euclid_N(const Poly& m, const Poly& M) {
  Poly r0 = M, s0{Rat(1)}, r1 = m, s1{};
  pnorm(r0);
  pnorm(r1);
  while (!r1.empty()) {
    Poly q, r2;
    pdivmod(r0, r1, q, r2);
    Poly s2 = psub(s0, pmul(q, s1));
    r0 = r1;
    s0 = s1;
    r1 = r2;
    s1 = s2;
  }
  if (pdeg(r0) != 0) throw ConfigError("moduli are not coprime");
  Poly N = pscale(s0, Rat(1) / r0[0]);
  if (pdeg(m) > 0 && pdeg(N) >= pdeg(m)) N = prem(N, m);
  return N;
}

using Mat = std::vector<std::vector<Rat>>;

inline Mat mmul(const Mat& a, const Mat& b) {
  size_t n = a.size(), k = b.size(), mcols = b.empty() ? 0 : b[0].size();
  Mat r(n, std::vector<Rat>(mcols));
  for (size_t i = 0; i < n; ++i)
    for (size_t t = 0; t < k; ++t) {
      if (a[i][t].is_zero()) continue;
      for (size_t j = 0; j < mcols; ++j) r[i][j] = r[i][j] + a[i][t] * b[t][j];
    }
  return r;
}

}  // namespace wino
