// xform_bf16.cu -- BF16 instantiations of the transform kernels (transforms_impl.cuh).
#include "transforms_impl.cuh"

namespace wino {
const InFn kInTableBF16[kTabM][kTabD] = WINO_TABLE(launch_in, WINO_BF16);
const OutFn kOutTableBF16[kTabM][kTabD] = WINO_TABLE(launch_out, WINO_BF16);
}  // namespace wino
