// xform.cu -- instantiations of the transform kernels (transforms_impl.cuh) for
// one (dtype, kind, m-range) part; build.py compiles this file 18 times with
//   -DWINO_XF_DT=<0 fp32 | 1 fp16 | 2 bf16>  -DWINO_XF_KIND=<0 input (K1) | 1 output (K4)>
//   -DWINO_XF_PART=<0: m = 2..5 | 1: m = 6..8 | 2: m = 9..12>
// so the (large, fully unrolled) instantiations compile in parallel.  Each unit
// defines one slice of the (m, domain) dispatch table read by transforms.cu.
#include "transforms_impl.cuh"

#if !defined(WINO_XF_DT) || !defined(WINO_XF_KIND) || !defined(WINO_XF_PART)
#error "compile xform.cu with -DWINO_XF_DT, -DWINO_XF_KIND and -DWINO_XF_PART (see build.py)"
#endif

namespace wino {
#if WINO_XF_KIND == 0
#define XF_FN launch_in
using XfT = InFn;
#else
#define XF_FN launch_out
using XfT = OutFn;
#endif
#define XF_CAT3(a, b, c, d) a##b##_##c##_##d
#define XF_NAME(k, d, p) XF_CAT3(kXf, k, d, p)

#if WINO_XF_PART == 0
extern const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows0][kTabD];
const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows0][kTabD] = {
    WINO_ROW(XF_FN, WINO_XF_DT, 2), WINO_ROW(XF_FN, WINO_XF_DT, 3), WINO_ROW(XF_FN, WINO_XF_DT, 4),
    WINO_ROW(XF_FN, WINO_XF_DT, 5)};
#elif WINO_XF_PART == 1
extern const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows1][kTabD];
const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows1][kTabD] = {
    WINO_ROW(XF_FN, WINO_XF_DT, 6), WINO_ROW(XF_FN, WINO_XF_DT, 7), WINO_ROW(XF_FN, WINO_XF_DT, 8)};
#else
extern const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows2][kTabD];
const XfT XF_NAME(WINO_XF_KIND, WINO_XF_DT, WINO_XF_PART)[kXfRows2][kTabD] = {
    WINO_ROW3(XF_FN, WINO_XF_DT, 9), WINO_ROW3(XF_FN, WINO_XF_DT, 10), WINO_ROW3(XF_FN, WINO_XF_DT, 11),
    WINO_ROW3(XF_FN, WINO_XF_DT, 12)};
#endif
}  // namespace wino
