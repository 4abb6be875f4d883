// xform_f32.cu -- F32 instantiations of the transform kernels (transforms_impl.cuh).
#include "transforms_impl.cuh"

namespace wino {
const InFn kInTableF32[kTabM][kTabD] = WINO_TABLE(launch_in, WINO_F32);
const OutFn kOutTableF32[kTabM][kTabD] = WINO_TABLE(launch_out, WINO_F32);
}  // namespace wino
