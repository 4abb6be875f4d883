"""ctypes loader for libwino.so (the C ABI declared in include/wino.h).

Argument marshalling only.  Fails loudly when the in-tree library is missing:
there is no fallback of any kind.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwino.so")

WINO_OK, WINO_E_ARG, WINO_E_CONFIG, WINO_E_RANGE, WINO_E_UNSUPPORTED, WINO_E_CUDA, WINO_E_WORKSPACE = range(7)
STATUS_NAMES = {0: "WINO_OK", 1: "WINO_E_ARG", 2: "WINO_E_CONFIG", 3: "WINO_E_RANGE", 4: "WINO_E_UNSUPPORTED",
                5: "WINO_E_CUDA", 6: "WINO_E_WORKSPACE"}
DTYPES = {"fp32": 0, "fp16": 1, "bf16": 2}
LAYOUTS = {"nchw": 0, "nhwc": 1}
LOWERINGS = {"subsolver": 0, "residue": 1}


class WinoModulus(ctypes.Structure):
    _fields_ = [("degree", ctypes.c_int32), ("num", ctypes.c_int64 * 5), ("den", ctypes.c_int64 * 5)]


class WinoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_I32 = ctypes.c_int32
_SIGS = {
    "wino_parse_moduli": (_I, [ctypes.c_char_p, ctypes.POINTER(WinoModulus), _I32, ctypes.POINTER(_I32)]),
    "wino_make_transforms": (_I, [ctypes.POINTER(WinoModulus), _I32, _I32, _I32, ctypes.POINTER(WinoModulus), _I32,
                                  _I, ctypes.POINTER(_P)]),
    "wino_algo_info": (_I, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                            ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(ctypes.c_double)]),
    "wino_algo_matrix": (_I, [_P, ctypes.c_char, _P, _P, _P]),
    "wino_algo_units": (_I, [_P, _P, _P, _P, _P, _P]),
    "wino_scale_transforms": (_I, [_P, ctypes.c_int32]),
    "wino_set_m_storage": (_I, [_P, ctypes.c_int32]),
    "wino_last_error": (ctypes.c_char_p, []),
    "wino_algo_destroy": (None, [_P]),
    "wino_conv2d_workspace": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, ctypes.POINTER(ctypes.c_size_t)]),
    "wino_conv2d": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P, ctypes.c_size_t, _P]),
    "wino_conv2d_host_io": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P, _P, ctypes.c_size_t, _P]),
    "wino_weight_transform": (_I, [_P, _I, _I, _P, _I, _P, _P]),
    "wino_input_transform": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P]),
    "wino_domain_gemm": (_I, [_P, _P, _I, _I, _I, _P, _I, _P, _P]),
    "wino_output_transform": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P]),
    "wino_conv1d_tiles": (_I, [_P, _P, ctypes.c_int64, _P, _I, _I, _P, _P]),
    "wino_conv2d_tiles_paper": (_I, [_P, _P, _I, ctypes.c_int64, _P, _I, _I, _I, _I, _P, _P]),
    "wino_error_stats_scratch": (ctypes.c_size_t, [_I, _I, _I, _I, _I]),
    "wino_error_stats": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "wino_direct_conv2d_f64": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P]),
    "wino_last_launch_count": (_I32, []),
}


def lib():
    """Load the in-tree libwino.so (build it with `python -m paper_1905_05233_b200.build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first "
                              "(python -m paper_1905_05233_b200.build); there is no fallback path")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status):
    if status != WINO_OK:
        msg = lib().wino_last_error()
        raise WinoError(status, msg.decode() if msg else "")
    return status
