// generator.cpp -- host-side exact CRT transform generator (Sec. 2.2).
//
//  * Toom-Cook sub-solver F_TC(d x d, d x d) in the paper's convention
//    (P:242-243): G^(TC) row_i = N_i [q_i^0 .. q_i^{d-1}]
//    with N_i = 1 / M_i(q_i); A^(TC) row_i = [q_i^0 .. q_i^{d-1}];
//    B^(TC) column_i = vec(M_i(a)); the pseudo-point column is vec(M(a)).
//  * Algorithm 1: G^W, A^W; linear moduli give unscaled Vandermonde
//    rows, degree-d moduli give G^(TC) G' and A^(TC) A', with A' having
//    n_o columns (reading A1 of DESIGN.md), infinity gives [0 .. 0 1].
//  * Algorithm 2: C = blockdiag(C_i), E_i = vec(R_M[a^k N_i M_i])
//    with N_i from the extended Euclidean algorithm (reading A2), zero row
//    appended to E iff infinity is used, B^W = [E C | vec M].
//  * Role assignment for Eq. (2) (reading A4): G := G^W, B := B^W, A := A^W.
//  * Residue lowering ("any suitable algorithm"): G_P = stacked
//    G' residue maps, B_P = [E | vec M], A_P = stacked A'; block products via
//    the matrices of multiplication by a^k modulo m_i.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

#include "algo.hpp"

namespace wino {

static const Rat kPaperPoints[9] = {Rat(0), Rat(-1), Rat(1), Rat::make(-1, 2), Rat(2),
                                    Rat::make(1, 2), Rat(-2), Rat::make(-1, 4), Rat(4)};

static std::string rat_str(const Rat& q) {
  auto i2s = [](i128 v) {
    bool neg = v < 0;
    if (neg) v = -v;
    std::string s;
    do {
      s.insert(s.begin(), char('0' + int(v % 10)));
      v /= 10;
    } while (v);
    return neg ? "-" + s : s;
  };
  return q.d == 1 ? i2s(q.n) : i2s(q.n) + "/" + i2s(q.d);
}

static std::string mod_str(const Modulus& m) {
  if (m.degree == 0) return "inf";
  if (m.degree == 1) return rat_str(m.root());
  std::string s;
  for (int k = m.degree; k >= 0; --k) {
    const Rat& c = m.poly[k];
    if (c.is_zero()) continue;
    std::string mono = k == 0 ? "" : (k == 1 ? "a" : "a^" + std::to_string(k));
    bool neg = c.n < 0;
    Rat ac = neg ? -c : c;
    std::string t = (!mono.empty() && ac == Rat(1)) ? mono : rat_str(ac) + (mono.empty() ? "" : "*" + mono);
    s += (neg ? "-" : (s.empty() ? "" : "+")) + t;
  }
  return s;
}

static bool has_rational_root2(const Poly& p) {  // monic degree 2
  Rat c = p[0], b = p[1];
  Rat disc = b * b - Rat(4) * c;
  if (disc.n < 0) return false;
  auto isq = [](i128 v) {
    long double f = std::sqrt((long double)v);
    i128 s = (i128)f;
    while (s * s > v) --s;
    while ((s + 1) * (s + 1) <= v) ++s;
    return s * s == v;
  };
  return isq(disc.n) && isq(disc.d);
}

// sub-solver matrices; rows/columns follow the point order.
static void toom_cook_sub(const std::vector<Modulus>& pts, int d, Mat& Gtc, Mat& Atc, Mat& Btc) {
  int n = 2 * d - 1;
  Poly Msub{Rat(1)};
  for (auto& q : pts)
    if (q.degree == 1) Msub = pmul(Msub, q.poly);
  Gtc.assign(n, std::vector<Rat>(d));
  Atc.assign(n, std::vector<Rat>(d));
  Btc.assign(n, std::vector<Rat>(n));
  for (int i = 0; i < n; ++i) {
    std::vector<Rat> col;
    if (pts[i].degree == 0) {
      Gtc[i][d - 1] = Rat(1);
      Atc[i][d - 1] = Rat(1);
      col = pvec(Msub, n);
    } else {
      Rat q = pts[i].root();
      Poly Mi = pquo(Msub, pts[i].poly);
      Rat Ni = Rat(1) / peval(Mi, q);
      Rat pw(1);
      for (int j = 0; j < d; ++j) {
        Gtc[i][j] = Ni * pw;
        Atc[i][j] = pw;
        pw = pw * q;
      }
      col = pvec(Mi, n);
    }
    for (int k = 0; k < n; ++k) Btc[k][i] = col[k];
  }
}

// d x ncols matrix whose column j is vec(R_m[a^j]).
static Mat residue_map(const Poly& m, int ncols) {
  int d = pdeg(m);
  Mat R(d, std::vector<Rat>(ncols));
  for (int j = 0; j < ncols; ++j) {
    auto v = pvec(prem(pmonomial(j), m), d);
    for (int i = 0; i < d; ++i) R[i][j] = v[i];
  }
  return R;
}

// column j = vec(R_m[a^{k+j}]): multiplication by a^k modulo m.
static Mat mult_matrix(const Poly& m, int k) {
  int d = pdeg(m);
  Mat R(d, std::vector<Rat>(d));
  for (int j = 0; j < d; ++j) {
    auto v = pvec(prem(pmonomial(k + j), m), d);
    for (int i = 0; i < d; ++i) R[i][j] = v[i];
  }
  return R;
}

static std::vector<Modulus> default_sub_points(int d) {
  std::vector<Modulus> out;
  for (int i = 0; i < 2 * d - 2; ++i) {
    Modulus q;
    q.degree = 1;
    q.poly = plinear(kPaperPoints[i]);
    out.push_back(q);
  }
  out.push_back(Modulus{});
  return out;
}

static void validate(const std::vector<Modulus>& mods, int m, int r, const std::vector<Modulus>* sub) {
  std::vector<std::string> v;
  int n_inf = 0;
  for (auto& q : mods) n_inf += q.degree == 0;
  if (n_inf > 1) v.push_back("pseudo-point inf appears more than once");
  if (n_inf == 1 && mods.back().degree != 0) v.push_back("pseudo-point inf must be the last modulus");
  int need = n_inf ? m + r - 2 : m + r - 1, have = 0;
  std::vector<const Modulus*> fin;
  for (auto& q : mods)
    if (q.degree > 0) fin.push_back(&q), have += q.degree;
  if (have != need)
    v.push_back("degree budget: sum deg = " + std::to_string(have) + ", need " + std::to_string(need));
  for (size_t i = 0; i < fin.size(); ++i) {
    if (fin[i]->degree == 2 && has_rational_root2(fin[i]->poly))
      v.push_back("modulus " + mod_str(*fin[i]) + " is reducible over Q");
    for (size_t j = i + 1; j < fin.size(); ++j)
      if (pdeg(pgcd(fin[i]->poly, fin[j]->poly)) > 0)
        v.push_back("moduli " + mod_str(*fin[i]) + " and " + mod_str(*fin[j]) + " are not coprime");
  }
  for (auto* q : fin) {
    if (q->degree < 2) continue;
    std::vector<Modulus> sp = sub ? *sub : default_sub_points(q->degree);
    if ((int)sp.size() != 2 * q->degree - 1) {
      v.push_back("modulus " + mod_str(*q) + ": sub-solver needs " + std::to_string(2 * q->degree - 1) +
                  " points, got " + std::to_string(sp.size()));
      continue;
    }
    int ninf = 0;
    bool dup = false;
    for (size_t i = 0; i < sp.size(); ++i) {
      if (sp[i].degree > 1) v.push_back("sub-solver points must be points or inf");
      ninf += sp[i].degree == 0;
      for (size_t j = i + 1; j < sp.size(); ++j)
        if (sp[i].degree == 1 && sp[j].degree == 1 && sp[i].poly == sp[j].poly) dup = true;
    }
    if (dup || ninf > 1) v.push_back("modulus " + mod_str(*q) + ": duplicate sub-solver points");
    else if (ninf == 1 && sp.back().degree != 0) v.push_back("modulus " + mod_str(*q) + ": inf must be the last sub-solver point");
  }
  if (!v.empty()) {
    std::string s;
    for (auto& e : v) s += e + "\n";
    throw ConfigError(s);
  }
}

float rat_to_f32(const Rat& q) {
  // Correctly rounded for |n| < 2^62, d < 2^31: the 64-bit-significand quotient
  // can never land on an fp32 rounding midpoint it is not equal to.
  if (iabs(q.n) >= ((i128)1 << 62) || q.d >= ((i128)1 << 31)) throw RangeError("entry too large for fp32 lowering");
  long double v = (long double)(long long)q.n / (long double)(long long)q.d;
  return (float)v;
}

wino_algo* generate(const std::vector<Modulus>& mods, int m, int r, const std::vector<Modulus>* sub,
                    wino_lowering lowering) {
  validate(mods, m, r, sub);
  auto* al = new wino_algo();
  try {
    al->m = m;
    al->r = r;
    al->nx = m + r - 1;
    al->mods = mods;
    al->lowering = lowering;
    bool has_inf = mods.back().degree == 0;
    std::vector<const Modulus*> fin;
    for (auto& q : mods)
      if (q.degree > 0) fin.push_back(&q);
    int mu = 0;
    for (auto& q : mods) mu += q.degree == 0 ? 1 : 2 * q.degree - 1;
    al->mu = mu;

    // ---- Algorithm 1
    Mat GW, AW;
    for (auto* q : fin) {
      int d = q->degree;
      if (d == 1) {
        Rat p = q->root(), pw(1);
        std::vector<Rat> g(r), a(m);
        for (int j = 0; j < std::max(r, m); ++j) {
          if (j < r) g[j] = pw;
          if (j < m) a[j] = pw;
          pw = pw * p;
        }
        GW.push_back(g);
        AW.push_back(a);
      } else {
        Mat Gtc, Atc, Btc;
        toom_cook_sub(sub ? *sub : default_sub_points(d), d, Gtc, Atc, Btc);
        for (auto& row : mmul(Gtc, residue_map(q->poly, r))) GW.push_back(row);
        for (auto& row : mmul(Atc, residue_map(q->poly, m))) AW.push_back(row);
      }
    }
    if (has_inf) {
      std::vector<Rat> g(r), a(m);
      g[r - 1] = Rat(1);
      a[m - 1] = Rat(1);
      GW.push_back(g);
      AW.push_back(a);
    }
    // ---- Algorithm 2
    Poly M{Rat(1)};
    for (auto* q : fin) M = pmul(M, q->poly);
    int degM = pdeg(M);
    int nrowE = degM + (has_inf ? 1 : 0);  // = nx
    // columns of E (all blocks), and the C blocks
    std::vector<std::vector<Rat>> Ecols;
    std::vector<Mat> Cblocks;
    for (auto* q : fin) {
      int d = q->degree;
      Poly Mi = pquo(M, q->poly);
      Poly Ni = ext_euclid_N(q->poly, Mi);
      Poly NiMi = pmul(Ni, Mi);
      for (int k = 0; k < d; ++k) {
        auto v = pvec(prem(pmul(pmonomial(k), NiMi), M), degM);
        if (has_inf) v.push_back(Rat());
        Ecols.push_back(v);
      }
      if (d == 1) {
        Cblocks.push_back(Mat{{Rat(1)}});
      } else {
        Mat Gtc, Atc, Btc;
        toom_cook_sub(sub ? *sub : default_sub_points(d), d, Gtc, Atc, Btc);
        int nc = 2 * d - 1;
        Mat Ci(d, std::vector<Rat>(nc));
        for (int j = 0; j < nc; ++j) {
          Poly bj(nc);
          for (int i = 0; i < nc; ++i) bj[i] = Btc[i][j];  // b_j(a)
          pnorm(bj);
          auto v = pvec(prem(bj, q->poly), d);
          for (int i = 0; i < d; ++i) Ci[i][j] = v[i];
        }
        Cblocks.push_back(Ci);
      }
    }
    int nE = (int)Ecols.size();
    Mat E(nrowE, std::vector<Rat>(nE));
    for (int j = 0; j < nE; ++j)
      for (int i = 0; i < nrowE; ++i) E[i][j] = Ecols[j][i];
    int Crow = 0, Ccol = 0;
    for (auto& b : Cblocks) Crow += (int)b.size(), Ccol += (int)b[0].size();
    Mat C(Crow, std::vector<Rat>(Ccol));
    for (int bi = 0, r0 = 0, c0 = 0; bi < (int)Cblocks.size(); ++bi) {
      auto& b = Cblocks[bi];
      for (size_t i = 0; i < b.size(); ++i)
        for (size_t j = 0; j < b[0].size(); ++j) C[r0 + i][c0 + j] = b[i][j];
      r0 += (int)b.size();
      c0 += (int)b[0].size();
    }
    Mat BW = mmul(E, C);
    std::vector<Rat> vM = pvec(M, degM + 1);
    if (has_inf)
      for (int i = 0; i < nrowE; ++i) BW[i].push_back(vM[i]);

    if (lowering == WINO_LOWER_SUBSOLVER) {
      al->G = GW;
      al->B = BW;
      al->A = AW;
      al->D = mu;
      al->units = mu * mu;
      for (int u = 0; u < al->units; ++u) {
        al->out_pt.push_back(u);
        al->in_pt.push_back(u);
        al->nterm.push_back(1);
        int a4[4] = {u, 0, 0, 0};
        Rat c4[4] = {Rat(1), Rat(), Rat(), Rat()};
        for (int j = 0; j < 4; ++j) al->ta.push_back(a4[j]), al->tcoef.push_back(c4[j]);
      }
    } else {
      // ---- residue lowering
      for (auto* q : fin)
        if (q->degree > 2) throw ConfigError("residue lowering supports moduli of degree <= 2");
      Mat GP, AP;
      struct Blk { int start, size; std::vector<Mat> phi; };
      std::vector<Blk> blocks;
      for (auto* q : fin) {
        Blk b{(int)GP.size(), q->degree, {}};
        for (auto& row : residue_map(q->poly, r)) GP.push_back(row);
        for (auto& row : residue_map(q->poly, m)) AP.push_back(row);
        for (int k = 0; k < q->degree; ++k) b.phi.push_back(mult_matrix(q->poly, k));
        blocks.push_back(b);
      }
      if (has_inf) {
        Blk b{(int)GP.size(), 1, {Mat{{Rat(1)}}}};
        std::vector<Rat> g(r), a(m);
        g[r - 1] = Rat(1);
        a[m - 1] = Rat(1);
        GP.push_back(g);
        AP.push_back(a);
        blocks.push_back(b);
      }
      Mat BP = E;
      if (has_inf)
        for (int i = 0; i < nrowE; ++i) BP[i].push_back(vM[i]);
      al->G = GP;
      al->B = BP;
      al->A = AP;
      int D = (int)GP.size();
      al->D = D;
      for (auto& I : blocks)
        for (auto& J : blocks)
          for (int k = 0; k < I.size; ++k)
            for (int l = 0; l < J.size; ++l)
              for (int kk = 0; kk < I.size; ++kk)
                for (int ll = 0; ll < J.size; ++ll) {
                  al->out_pt.push_back((I.start + k) * D + (J.start + l));
                  al->in_pt.push_back((I.start + kk) * D + (J.start + ll));
                  int nt = 0;
                  int a4[4] = {0, 0, 0, 0};
                  Rat c4[4];
                  for (int a = 0; a < I.size; ++a)
                    for (int b = 0; b < J.size; ++b) {
                      Rat cf = I.phi[a][kk][k] * J.phi[b][ll][l];
                      if (cf.is_zero()) continue;
                      a4[nt] = (I.start + a) * D + (J.start + b);
                      c4[nt] = cf;
                      ++nt;
                    }
                  al->nterm.push_back(nt);
                  for (int j = 0; j < 4; ++j) al->ta.push_back(a4[j]), al->tcoef.push_back(c4[j]);
                }
      al->units = (int)al->out_pt.size();
    }
    if (al->D > kMaxDomain) throw ConfigError("domain size > 16 unsupported");
    if (al->units > kMaxUnits) throw ConfigError("more than 256 GEMM units unsupported");

    // ---- fp32 lowering into kernel parameter blocks
    XformParams& xp = al->xp;
    std::memset(&xp, 0, sizeof(xp));
    xp.m = m;
    xp.nx = al->nx;
    xp.D = al->D;
    for (int i = 0; i < al->D; ++i) {
      for (int j = 0; j < al->nx; ++j) xp.BT[i][j] = rat_to_f32(al->B[j][i]);
      for (int j = 0; j < r; ++j) xp.G[i][j] = rat_to_f32(al->G[i][j]);
      for (int j = 0; j < m; ++j) xp.AT[j][i] = rat_to_f32(al->A[i][j]);
    }
    UnitTerms& ut = al->ut;
    std::memset(&ut, 0, sizeof(ut));
    ut.units = al->units;
    for (int u = 0; u < al->units; ++u) {
      ut.nterm[u] = (unsigned char)al->nterm[u];
      for (int j = 0; j < 4; ++j) {
        ut.a[u][j] = (unsigned char)al->ta[4 * u + j];
        ut.coef[u][j] = rat_to_f32(al->tcoef[4 * u + j]);
      }
    }
    GemmSched& gs = al->gs;
    std::memset(&gs, 0, sizeof(gs));
    gs.Q = al->D * al->D;
    gs.npairs = al->units;
    int idx = 0;
    for (int p = 0; p < gs.Q; ++p) {
      gs.off[p] = (short)idx;
      for (int u = 0; u < al->units; ++u)
        if (al->out_pt[u] == p) {
          gs.in_pt[idx] = (unsigned char)al->in_pt[u];
          gs.slab[idx] = (unsigned char)u;
          ++idx;
        }
    }
    gs.off[gs.Q] = (short)idx;
  } catch (...) {
    delete al;
    throw;
  }
  return al;
}

// ---------------------------------------------------------------- parsing

static std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t"), b = s.find_last_not_of(" \t");
  return a == std::string::npos ? "" : s.substr(a, b - a + 1);
}

static Rat parse_rat(const std::string& s) {
  if (s.empty()) throw ConfigError("empty number");
  size_t slash = s.find('/');
  auto toi = [](const std::string& t) -> long long {
    if (t.empty()) throw ConfigError("bad number");
    size_t pos = 0;
    long long v = std::stoll(t, &pos);
    if (pos != t.size()) throw ConfigError("bad number '" + t + "'");
    return v;
  };
  if (slash == std::string::npos) return Rat(toi(s));
  return Rat::make(toi(s.substr(0, slash)), toi(s.substr(slash + 1)));
}

static Poly parse_poly(std::string s) {
  s.erase(std::remove(s.begin(), s.end(), ' '), s.end());
  if (s.empty()) throw ConfigError("empty polynomial");
  std::vector<Rat> c(8);
  size_t i = 0;
  while (i < s.size()) {
    int sign = 1;
    if (s[i] == '+' || s[i] == '-') sign = s[i] == '-' ? -1 : 1, ++i;
    size_t j = i;
    while (j < s.size() && (isdigit((unsigned char)s[j]) || s[j] == '/')) ++j;
    std::string num = s.substr(i, j - i);
    i = j;
    if (i < s.size() && s[i] == '*') ++i;
    int k = 0;
    bool mono = false;
    if (i < s.size() && s[i] == 'a') {
      mono = true;
      ++i;
      k = 1;
      if (i < s.size() && s[i] == '^') {
        ++i;
        size_t e = i;
        while (e < s.size() && isdigit((unsigned char)s[e])) ++e;
        if (e == i) throw ConfigError("bad exponent in '" + s + "'");
        k = std::stoi(s.substr(i, e - i));
        i = e;
      }
    }
    if (num.empty() && !mono) throw ConfigError("cannot parse polynomial '" + s + "'");
    if (k > 7) throw ConfigError("polynomial degree too large");
    Rat cf = num.empty() ? Rat(1) : parse_rat(num);
    c[k] = c[k] + (sign < 0 ? -cf : cf);
  }
  pnorm(c);
  return c;
}

std::vector<Modulus> parse_moduli(const std::string& spec) {
  std::vector<Modulus> out;
  std::stringstream ss(spec);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    tok = trim(tok);
    std::string low = tok;
    std::transform(low.begin(), low.end(), low.begin(), ::tolower);
    Modulus q;
    if (low == "inf" || low == "infinity") {
      q.degree = 0;
    } else if (tok.find('a') != std::string::npos) {
      Poly p = pmonic(parse_poly(tok));
      if (pdeg(p) < 1) throw ConfigError("modulus '" + tok + "' has degree < 1");
      q.degree = pdeg(p);
      q.poly = p;
    } else {
      q.degree = 1;
      q.poly = plinear(parse_rat(tok));
    }
    out.push_back(q);
  }
  return out;
}

}  // namespace wino
