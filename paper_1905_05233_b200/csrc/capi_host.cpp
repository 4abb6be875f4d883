// capi_host.cpp -- host-only C-ABI entry points of libwino.so (include/wino.h):
// parsing, transform generation, introspection.  Never touches CUDA.
#include <cstring>
#include <string>

#include "algo.hpp"

namespace wino {
static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
}  // namespace wino

using namespace wino;

static bool to_internal(const wino_modulus& in, Modulus& out, std::string& err) {
  if (in.degree < 0 || in.degree > 4) {
    err = "modulus degree must be 0..4";
    return false;
  }
  out.degree = in.degree;
  if (in.degree == 0) return true;
  for (int k = 0; k <= (in.degree == 1 ? 0 : in.degree); ++k)
    if (in.den[k] == 0) {
      err = "zero denominator";
      return false;
    }
  if (in.degree == 1) {
    out.poly = plinear(Rat::make(in.num[0], in.den[0]));
    return true;
  }
  Poly p(in.degree + 1);
  for (int k = 0; k <= in.degree; ++k) p[k] = Rat::make(in.num[k], in.den[k]);
  pnorm(p);
  if (pdeg(p) != in.degree) {
    err = "leading coefficient is zero";
    return false;
  }
  out.poly = pmonic(p);
  return true;
}

static void to_external(const Modulus& in, wino_modulus& out) {
  std::memset(&out, 0, sizeof(out));
  out.degree = in.degree;
  for (int k = 0; k < 5; ++k) out.den[k] = 1;
  if (in.degree == 1) {
    Rat p = in.root();
    out.num[0] = (int64_t)p.n;
    out.den[0] = (int64_t)p.d;
  } else if (in.degree >= 2) {
    for (int k = 0; k <= in.degree; ++k) {
      out.num[k] = (int64_t)in.poly[k].n;
      out.den[k] = (int64_t)in.poly[k].d;
    }
  }
}

extern "C" {

const char* wino_last_error(void) { return g_last_error.c_str(); }

wino_status wino_parse_moduli(const char* spec, wino_modulus* mods, int32_t cap, int32_t* n) {
  if (!spec || !n || (cap > 0 && !mods) || cap < 0) {
    set_last_error("wino_parse_moduli: bad argument");
    return WINO_E_ARG;
  }
  try {
    auto v = parse_moduli(spec);
    for (auto& q : v)
      if (q.degree > 4) throw ConfigError("modulus degree > 4 unsupported");
    *n = (int32_t)v.size();
    if ((int32_t)v.size() > cap) {
      set_last_error("wino_parse_moduli: capacity too small");
      return WINO_E_ARG;
    }
    for (size_t i = 0; i < v.size(); ++i) to_external(v[i], mods[i]);
    return WINO_OK;
  } catch (const std::exception& e) {
    set_last_error(std::string("wino_parse_moduli: ") + e.what());
    return WINO_E_CONFIG;
  }
}

wino_status wino_make_transforms(const wino_modulus* mods, int32_t n_mods, int32_t m, int32_t r,
                                 const wino_modulus* sub_points, int32_t n_sub, wino_lowering lowering,
                                 wino_algo** out) {
  if (!mods || n_mods <= 0 || !out || (n_sub > 0 && !sub_points) || n_sub < 0 ||
      (lowering != WINO_LOWER_SUBSOLVER && lowering != WINO_LOWER_RESIDUE)) {
    set_last_error("wino_make_transforms: bad argument");
    return WINO_E_ARG;
  }
  *out = nullptr;
  if (r != 3 || m < 2 || m > 12) {
    set_last_error("wino_make_transforms: only r = 3 and 2 <= m <= 12 are supported");
    return WINO_E_UNSUPPORTED;
  }
  std::vector<Modulus> v(n_mods), sp(n_sub);
  std::string err;
  for (int i = 0; i < n_mods; ++i)
    if (!to_internal(mods[i], v[i], err)) {
      set_last_error("wino_make_transforms: " + err);
      return WINO_E_ARG;
    }
  for (int i = 0; i < n_sub; ++i)
    if (!to_internal(sub_points[i], sp[i], err)) {
      set_last_error("wino_make_transforms: " + err);
      return WINO_E_ARG;
    }
  try {
    *out = generate(v, m, r, n_sub > 0 ? &sp : nullptr, lowering);
    int mu = (*out)->mu;
    if (mu > kMaxDomain) {
      wino_algo_destroy(*out);
      *out = nullptr;
      set_last_error("wino_make_transforms: mu > 16 unsupported");
      return WINO_E_UNSUPPORTED;
    }
    return WINO_OK;
  } catch (const RangeError& e) {
    set_last_error(std::string("wino_make_transforms: ") + e.what());
    return WINO_E_RANGE;
  } catch (const std::exception& e) {
    set_last_error(std::string("wino_make_transforms: ") + e.what());
    return WINO_E_CONFIG;
  }
}

wino_status wino_algo_info(const wino_algo* al, int32_t* m, int32_t* mu, int32_t* nx, int32_t* domain,
                           int32_t* units, double* ratio_2d) {
  if (!al) {
    set_last_error("wino_algo_info: NULL algo");
    return WINO_E_ARG;
  }
  if (m) *m = al->m;
  if (mu) *mu = al->mu;
  if (nx) *nx = al->nx;
  if (domain) *domain = al->D;
  if (units) *units = al->units;
  if (ratio_2d) *ratio_2d = double(al->mu) * al->mu / (double(al->m) * al->m);
  return WINO_OK;
}

wino_status wino_algo_matrix(const wino_algo* al, char which, int64_t* num, int64_t* den, float* f32) {
  if (!al) {
    set_last_error("wino_algo_matrix: NULL algo");
    return WINO_E_ARG;
  }
  const Mat* M = which == 'G' ? &al->G : which == 'B' ? &al->B : which == 'A' ? &al->A : nullptr;
  if (!M) {
    set_last_error("wino_algo_matrix: which must be 'G', 'B' or 'A'");
    return WINO_E_ARG;
  }
  size_t k = 0;
  for (auto& row : *M)
    for (auto& q : row) {
      if (num) num[k] = (int64_t)q.n;
      if (den) den[k] = (int64_t)q.d;
      if (f32) f32[k] = rat_to_f32(q);
      ++k;
    }
  return WINO_OK;
}

wino_status wino_algo_units(const wino_algo* al, int32_t* out_pt, int32_t* in_pt, int32_t* nterm, int32_t* a,
                            double* coef) {
  if (!al) {
    set_last_error("wino_algo_units: NULL algo");
    return WINO_E_ARG;
  }
  for (int u = 0; u < al->units; ++u) {
    if (out_pt) out_pt[u] = al->out_pt[u];
    if (in_pt) in_pt[u] = al->in_pt[u];
    if (nterm) nterm[u] = al->nterm[u];
    for (int j = 0; j < 4; ++j) {
      if (a) a[4 * u + j] = al->ta[4 * u + j];
      if (coef) coef[4 * u + j] = (double)(long double)al->tcoef[4 * u + j].n / (double)(long double)al->tcoef[4 * u + j].d;
    }
  }
  return WINO_OK;
}

void wino_algo_destroy(wino_algo* al) { delete al; }

// Power-of-two balancing of the Winograd points (include/wino.h, S1):
// B column i *= 2^-s_i, A row i *= 2^s_i, s_i = floor(floor(log2(max|B[:,i]| /
// max|A[i,:]|)) / 2).  Exact; re-lowers the fp32 kernel parameters.
static int floor_log2(const Rat& r) {   // r > 0
  int e = 0;
  Rat two = Rat(2), half = Rat::make(1, 2), p = Rat(1);
  auto lt = [](const Rat& a, const Rat& b) { return (a - b).n < 0; };
  auto le = [&](const Rat& a, const Rat& b) { return !lt(b, a); };
  while (lt(r, p)) p = p * half, --e;            // now p <= r (or it was already)
  while (le(p * two, r)) p = p * two, ++e;       // now p <= r < 2p
  return e;
}

wino_status wino_scale_transforms(wino_algo* al, int32_t mode) {
  if (!al) return set_last_error("wino_scale_transforms: NULL algo"), WINO_E_ARG;
  if (mode == WINO_SCALE_NONE) return WINO_OK;
  if (mode != WINO_SCALE_POW2_BALANCE) return set_last_error("wino_scale_transforms: bad mode"), WINO_E_ARG;
  if (al->lowering != WINO_LOWER_SUBSOLVER)
    return set_last_error("wino_scale_transforms: the SUBSOLVER lowering only"), WINO_E_UNSUPPORTED;
  if (al->scaled) return set_last_error("wino_scale_transforms: already scaled"), WINO_E_ARG;
  try {
    const int D = al->D;
    for (int i = 0; i < D; ++i) {
      Rat bmax(0), amax(0);
      auto absr = [](const Rat& q) { return q.n < 0 ? -q : q; };
      auto gt = [](const Rat& a, const Rat& b) { return (a - b).n > 0; };
      for (size_t j = 0; j < al->B.size(); ++j)
        if (gt(absr(al->B[j][i]), bmax)) bmax = absr(al->B[j][i]);
      for (size_t k = 0; k < al->A[i].size(); ++k)
        if (gt(absr(al->A[i][k]), amax)) amax = absr(al->A[i][k]);
      if (bmax.is_zero() || amax.is_zero()) continue;
      const int e = floor_log2(bmax / amax);
      const int s = e >= 0 ? e / 2 : -((-e + 1) / 2);   // floor(e / 2)
      Rat f(1);
      for (int t = 0; t < (s < 0 ? -s : s); ++t) f = f * Rat(2);
      if (s < 0) f = Rat(1) / f;
      for (size_t j = 0; j < al->B.size(); ++j) al->B[j][i] = al->B[j][i] / f;
      for (size_t k = 0; k < al->A[i].size(); ++k) al->A[i][k] = al->A[i][k] * f;
    }
    for (int i = 0; i < D; ++i) {
      for (int j = 0; j < al->nx; ++j) al->xp.BT[i][j] = rat_to_f32(al->B[j][i]);
      for (int j = 0; j < al->m; ++j) al->xp.AT[j][i] = rat_to_f32(al->A[i][j]);
    }
    al->scaled = true;
  } catch (const std::exception& ex) {
    set_last_error(std::string("wino_scale_transforms: ") + ex.what());
    return WINO_E_RANGE;
  }
  return WINO_OK;
}

wino_status wino_set_m_storage(wino_algo* al, int32_t mode) {
  if (!al) return set_last_error("wino_set_m_storage: NULL algo"), WINO_E_ARG;
  if (mode != WINO_M_FP32 && mode != WINO_M_DTYPE) return set_last_error("wino_set_m_storage: bad mode"), WINO_E_ARG;
  al->m_store = mode;
  return WINO_OK;
}

}  // extern "C"
