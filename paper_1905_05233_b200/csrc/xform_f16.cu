// xform_f16.cu -- F16 instantiations of the transform kernels (transforms_impl.cuh).
#include "transforms_impl.cuh"

namespace wino {
const InFn kInTableF16[kTabM][kTabD] = WINO_TABLE(launch_in, WINO_F16);
const OutFn kOutTableF16[kTabM][kTabD] = WINO_TABLE(launch_out, WINO_F16);
}  // namespace wino
