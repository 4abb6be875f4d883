// transforms.cu -- the three CUDA-core stages of the Winograd layer
// (Eq. 2: Y = A^T [(G g G^T) (.) (B^T d B)] A):
//   K2 weight transform  U_u[k][c] = rd(slab_u(G g_{k,c} G^T))       (A1)
//   K1 input transform   V_q[t][c] = rd((B^T d_{t,c} B)_q)           (A2)
//   K4 output transform  y[n,k,..] = rd(A^T M_{t,k} A), ragged-clipped (A4)
// All arithmetic is fp32 with the fp32-lowered exact matrices; rounding to the
// storage dtype happens once per stored tensor (the "pipeline" model).
#include <string>

#include "transforms_impl.cuh"

namespace wino {

// table slices of xform.cu: kXf<kind>_<dtype>_<part>, part 0: m = 2..5, 1: 6..8, 2: 9..12
#define XF_DECL(k, d)                                     \
  extern const XfT##k kXf##k##_##d##_0[kXfRows0][kTabD]; \
  extern const XfT##k kXf##k##_##d##_1[kXfRows1][kTabD]; \
  extern const XfT##k kXf##k##_##d##_2[kXfRows2][kTabD];
using XfT0 = InFn;
using XfT1 = OutFn;
XF_DECL(0, 0) XF_DECL(0, 1) XF_DECL(0, 2) XF_DECL(1, 0) XF_DECL(1, 1) XF_DECL(1, 2)
#undef XF_DECL
#define XF_PICK(k, d) (m <= 5 ? kXf##k##_##d##_0[m - 2][doff] : m <= 8 ? kXf##k##_##d##_1[m - 6][doff] : kXf##k##_##d##_2[m - 9][doff])
static InFn in_fn_(int dt, int m, int doff) {
  return dt == WINO_F32 ? XF_PICK(0, 0) : dt == WINO_F16 ? XF_PICK(0, 1) : XF_PICK(0, 2);
}
static OutFn out_fn_(int dt, int m, int doff) {
  return dt == WINO_F32 ? XF_PICK(1, 0) : dt == WINO_F16 ? XF_PICK(1, 1) : XF_PICK(1, 2);
}
#undef XF_PICK

// (m, D) with compiled transform kernels (WINO_TABLE)
static bool md_ok(const wino_algo* al) {
  const int doff = al->D - al->m - 2;
  return al->m >= 2 && al->m <= 12 && doff >= 0 && doff < kTabD && in_fn_(WINO_BF16, al->m, doff) != nullptr;
}

template <int DT, int D>
static void launch_wpts(const void* w, int K, int C, int Cp, const XformParams& xp, void* U, size_t plane,
                        cudaStream_t st) {
  using TT = typename DType<DT>::T;
  weight_transform_points<DT, D><<<dim3(Cp / 64, (K + 3) / 4), dim3(32, 4), 0, st>>>((const TT*)w, K, C, Cp, xp,
                                                                                    (TT*)U, plane);
}
template <int DT>
static bool weight_points(int D, const void* w, int K, int C, int Cp, const XformParams& xp, void* U, size_t plane,
                          cudaStream_t st) {
  switch (D) {
    case 4: launch_wpts<DT, 4>(w, K, C, Cp, xp, U, plane, st); return true;
    case 5: launch_wpts<DT, 5>(w, K, C, Cp, xp, U, plane, st); return true;
    case 6: launch_wpts<DT, 6>(w, K, C, Cp, xp, U, plane, st); return true;
    case 7: launch_wpts<DT, 7>(w, K, C, Cp, xp, U, plane, st); return true;
    case 8: launch_wpts<DT, 8>(w, K, C, Cp, xp, U, plane, st); return true;
    case 9: launch_wpts<DT, 9>(w, K, C, Cp, xp, U, plane, st); return true;
    case 10: launch_wpts<DT, 10>(w, K, C, Cp, xp, U, plane, st); return true;
    case 11: launch_wpts<DT, 11>(w, K, C, Cp, xp, U, plane, st); return true;
    case 12: launch_wpts<DT, 12>(w, K, C, Cp, xp, U, plane, st); return true;
    case 13: launch_wpts<DT, 13>(w, K, C, Cp, xp, U, plane, st); return true;
    case 14: launch_wpts<DT, 14>(w, K, C, Cp, xp, U, plane, st); return true;
    case 15: launch_wpts<DT, 15>(w, K, C, Cp, xp, U, plane, st); return true;
    case 16: launch_wpts<DT, 16>(w, K, C, Cp, xp, U, plane, st); return true;
    default: return false;
  }
}

wino_status run_weight_transform(const void* w, int K, int C, const wino_algo* al, wino_dtype dt, void* U,
                                 cudaStream_t st) {
  Geo g = make_geo(al, 1, C, 3, 3, K, 1, dt);
  size_t plane = (size_t)g.S * K * g.Cp;
  if (al->lowering == WINO_LOWER_SUBSOLVER && al->units == al->D * al->D) {
    // units are the D x D Winograd points in row-major order (identity schedule)
    const bool ok = dt == WINO_F32   ? weight_points<WINO_F32>(al->D, w, K, C, g.Cp, al->xp, U, plane, st)
                    : dt == WINO_F16 ? weight_points<WINO_F16>(al->D, w, K, C, g.Cp, al->xp, U, plane, st)
                                     : weight_points<WINO_BF16>(al->D, w, K, C, g.Cp, al->xp, U, plane, st);
    if (ok) {
      WINO_LAUNCH_CHECK();
      return WINO_OK;
    }
  }
  dim3 grid((g.Cp + 127) / 128, K);
  switch (dt) {
    case WINO_F32:
      weight_transform_kernel<WINO_F32><<<grid, 128, 0, st>>>((const float*)w, K, C, g.Cp, al->xp, al->ut,
                                                              (float*)U, plane);
      break;
    case WINO_F16:
      weight_transform_kernel<WINO_F16><<<grid, 128, 0, st>>>((const __half*)w, K, C, g.Cp, al->xp, al->ut,
                                                              (__half*)U, plane);
      break;
    case WINO_BF16:
      weight_transform_kernel<WINO_BF16><<<grid, 128, 0, st>>>((const __nv_bfloat16*)w, K, C, g.Cp, al->xp,
                                                               al->ut, (__nv_bfloat16*)U, plane);
      break;
  }
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

wino_status run_input_transform(const void* x, int N, int C, int H, int W, int pad, const wino_algo* al,
                                wino_dtype dt, wino_layout layout, void* V, cudaStream_t st) {
  if ((layout != WINO_NCHW && layout != WINO_NHWC) || !md_ok(al)) {
    set_last_error("input transform: unsupported layout / (m, domain)");
    return WINO_E_UNSUPPORTED;
  }
  Geo g = make_geo(al, N, C, H, W, 1, pad, dt);
  const size_t qstride = (size_t)128 * g.CBW;   // blocked V: adjacent point blocks (geometry.hpp)
  InArgs a{x, C, H, W, pad, g.th, g.tw, g.Cp, N, (int)layout, &al->xp, V, qstride, (size_t)g.Q * g.TB * 128 * g.Cp, st};
  in_fn_(dt, al->m, al->D - al->m - 2)(a);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

wino_status run_output_transform(const void* Mw, int N, int K, int H, int W, int pad, const wino_algo* al,
                                 wino_dtype dt, wino_layout layout, void* y, cudaStream_t st, int t0, int nT,
                                 int Tpm, int disc) {
  if ((layout != WINO_NCHW && layout != WINO_NHWC) || !md_ok(al)) {
    set_last_error("output transform: unsupported layout / (m, domain)");
    return WINO_E_UNSUPPORTED;
  }
  Geo g = make_geo(al, N, 1, H, W, K, pad, dt);
  OutArgs a{Mw, K, g.Ho, g.Wo, g.th, g.tw, g.T, nT < 0 ? g.Tp : Tpm, (int)layout, &al->xp, y, st};
  a.t0 = t0, a.nT = nT, a.disc = disc;
  a.m16 = m_in_dtype(al, dt) ? 1 : 0;
  out_fn_(dt, al->m, al->D - al->m - 2)(a);
  WINO_LAUNCH_CHECK();
  return WINO_OK;
}

}  // namespace wino
