// algo.hpp -- internal definition of the opaque wino_algo handle and the
// kernel parameter blocks derived from it.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/wino.h"
#include "exact.hpp"

namespace wino {

constexpr int kMaxDomain = 16;   // mu (or n_x) per dimension
constexpr int kMaxNx = 14;       // m + 2, m <= 12
constexpr int kMaxM = 12;
constexpr int kMaxUnits = 256;   // GEMM units per 2D tile

struct Modulus {
  int degree = 0;  // 0 = infinity
  Poly poly;       // monic (linear: a - p)
  Rat root() const { return -poly[0]; }
};

// fp32-lowered transform matrices of the selected lowering, passed by value
// to the transform kernels (lives in the kernel-parameter constant bank).
struct XformParams {
  int m, nx, D;
  float BT[kMaxDomain][kMaxNx];  // D x nx : input transform B^T
  float G[kMaxDomain][3];        // D x 3  : kernel transform
  float AT[kMaxM][kMaxDomain];   // m x D  : output transform A^T
};

// Weight-slab construction of the residue lowering (identity for SUBSOLVER).
struct UnitTerms {
  int units;
  unsigned char nterm[kMaxUnits];
  unsigned char a[kMaxUnits][4];   // row-major index into the D x D residue domain
  float coef[kMaxUnits][4];
};

// GEMM schedule: output point p accumulates pairs [off[p], off[p+1]).
struct GemmSched {
  int Q;        // output points
  int npairs;
  short off[kMaxDomain * kMaxDomain + 1];
  unsigned char in_pt[kMaxUnits];
  unsigned char slab[kMaxUnits];
};

}  // namespace wino

struct wino_algo {
  int m = 0, r = 3, nx = 0, mu = 0, D = 0, units = 0;
  wino_lowering lowering = WINO_LOWER_SUBSOLVER;
  bool scaled = false;   // wino_scale_transforms applied
  int m_store = 0;       // wino_set_m_storage: 0 = fp32 M (reading R1), 1 = M in the 16-bit layer dtype (M3)
  std::vector<wino::Modulus> mods;
  wino::Mat G, B, A;  // exact, selected lowering: G D x r, B nx x D, A D x m
  std::vector<int> out_pt, in_pt, nterm, ta;
  std::vector<wino::Rat> tcoef;
  wino::XformParams xp;
  wino::UnitTerms ut;
  wino::GemmSched gs;
};

namespace wino {
// generator.cpp
wino_algo* generate(const std::vector<Modulus>& mods, int m, int r, const std::vector<Modulus>* sub,
                    wino_lowering lowering);  // throws ConfigError / RangeError
std::vector<Modulus> parse_moduli(const std::string& spec);
float rat_to_f32(const Rat& q);
void set_last_error(const std::string& s);
}  // namespace wino
