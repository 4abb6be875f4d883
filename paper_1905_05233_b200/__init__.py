"""B200-native (sm_100a) Winograd convolution with CRT-generated transforms
(arXiv 1905.05233): exact host generator + CUDA kernels behind the C ABI of
include/wino.h, with this thin binding on top."""
from ._lib import WinoError, lib  # noqa: F401
from .api import (WinoAlgo, alloc_workspace, geometry, summary, wino_conv1d_tiles, wino_conv2d,
                  wino_conv2d_tiles_paper,  # noqa: F401
                  wino_conv2d_host_io, wino_conv2d_workspace, wino_direct_conv2d_f64, wino_domain_gemm,
                  wino_error_stats, wino_input_transform, wino_last_launch_count, wino_output_transform,
                  wino_parse_moduli, wino_weight_transform, v_from_dense, v_to_dense)
