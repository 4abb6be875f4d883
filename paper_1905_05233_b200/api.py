"""Thin Python binding over libwino.so (include/wino.h), same names as the C ABI.

PyTorch provides device memory and the current CUDA stream only; every step of
the path runs in the library's CUDA kernels.  Functions raise WinoError on any
non-OK status; there is no CPU fallback.
"""
import ctypes
from fractions import Fraction

import numpy as np
import torch

from ._lib import DTYPES, LAYOUTS, LOWERINGS, WinoError, WinoModulus, check, lib

_TORCH_DT = {torch.float32: "fp32", torch.float16: "fp16", torch.bfloat16: "bf16"}
TORCH_OF = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}


def _dt(t):
    try:
        return DTYPES[_TORCH_DT[t.dtype]]
    except KeyError:
        raise WinoError(1, f"unsupported dtype {t.dtype}")


def _stream(stream=None, device=None):
    """The stream the library launches on: `stream`, else the current stream of
    `device` (the tensors' device, not whichever device happens to be current)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _on_stream(stream, *tensors):
    """Allocations made on the current stream but used on another `stream` must
    not be recycled by the caching allocator before that stream's kernels ran."""
    if stream is None:
        return
    cur = torch.cuda.current_stream(stream.device)
    if stream.cuda_stream != cur.cuda_stream:
        for t in tensors:
            if t is not None and t.is_cuda:
                t.record_stream(stream)


def _check_out(out, shape, dtype, device):
    if tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != device or not out.is_contiguous():
        raise WinoError(1, f"out must be a contiguous {dtype} tensor of shape {tuple(shape)} on {device}; "
                           f"got {out.dtype} {tuple(out.shape)} on {out.device}"
                           f"{'' if out.is_contiguous() else ' (non-contiguous)'}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def wino_parse_moduli(spec):
    buf = (WinoModulus * 64)()
    n = ctypes.c_int32()
    check(lib().wino_parse_moduli(spec.encode(), buf, 64, ctypes.byref(n)))
    return list(buf[:n.value])


def _moduli_array(moduli):
    if isinstance(moduli, str):
        moduli = wino_parse_moduli(moduli)
    arr = (WinoModulus * len(moduli))()
    for i, m in enumerate(moduli):
        arr[i] = m
    return arr, len(moduli)


class WinoAlgo:
    """Owning handle of a generated algorithm (wino_make_transforms)."""

    def __init__(self, moduli, m, r=3, sub_points=None, lowering="subsolver"):
        self._h = None
        mods, n = _moduli_array(moduli)
        if sub_points is not None:
            sub, ns = _moduli_array(sub_points)
        else:
            sub, ns = None, 0
        h = ctypes.c_void_p()
        check(lib().wino_make_transforms(mods, n, m, r, sub, ns, LOWERINGS[lowering], ctypes.byref(h)))
        self._h = h
        self.spec = moduli if isinstance(moduli, str) else None
        self.lowering = lowering
        self.m_store = "fp32"
        vals = [ctypes.c_int32() for _ in range(5)]
        ratio = ctypes.c_double()
        check(lib().wino_algo_info(h, *[ctypes.byref(v) for v in vals], ctypes.byref(ratio)))
        self.m, self.mu, self.nx, self.domain, self.units = (v.value for v in vals)
        self.ratio_2d = ratio.value

    @property
    def handle(self):
        return self._h

    def matrix(self, which):
        """(exact Fraction matrix, fp32 numpy matrix) of 'G', 'B' or 'A'."""
        rows, cols = {"G": (self.domain, 3), "B": (self.nx, self.domain), "A": (self.domain, self.m)}[which]
        num = np.zeros(rows * cols, np.int64)
        den = np.zeros(rows * cols, np.int64)
        f32 = np.zeros(rows * cols, np.float32)
        check(lib().wino_algo_matrix(self._h, which.encode(), num.ctypes.data, den.ctypes.data, f32.ctypes.data))
        exact = [[Fraction(int(num[i * cols + j]), int(den[i * cols + j])) for j in range(cols)] for i in range(rows)]
        return exact, f32.reshape(rows, cols)

    def scale(self, mode="pow2"):
        """Power-of-two point balancing (wino_scale_transforms, [Vincent17] per P:607)."""
        check(lib().wino_scale_transforms(self._h, {"none": 0, "pow2": 1}[mode]))
        return self

    def set_m_storage(self, mode="dtype"):
        """Where the channel sum M lives between K3 and K4 (wino_set_m_storage):
        "fp32" (reading R1, default) or "dtype" (reading M3: the fp32
        accumulator rounded once to the layer's 16-bit dtype; fp32 layers and
        tiles beyond 8x8 keep fp32)."""
        check(lib().wino_set_m_storage(self._h, {"fp32": 0, "dtype": 1}[mode]))
        self.m_store = mode
        return self

    def unit_table(self):
        u = self.units
        out_pt, in_pt, nterm = (np.zeros(u, np.int32) for _ in range(3))
        a = np.zeros((u, 4), np.int32)
        coef = np.zeros((u, 4), np.float64)
        check(lib().wino_algo_units(self._h, out_pt.ctypes.data, in_pt.ctypes.data, nterm.ctypes.data,
                                    a.ctypes.data, coef.ctypes.data))
        return out_pt, in_pt, nterm, a, coef

    def close(self):
        if self._h is not None:
            lib().wino_algo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------- 2D layer


def wino_conv2d_workspace(algo, N, C, H, W, K, pad=1, dtype="bf16", layout="nchw"):
    b = ctypes.c_size_t()
    check(lib().wino_conv2d_workspace(algo.handle, N, C, H, W, K, pad, DTYPES[dtype], LAYOUTS[layout],
                                      ctypes.byref(b)))
    return b.value


def alloc_workspace(nbytes, device="cuda"):
    """Device workspace, 1024-byte aligned (the TMA/UMMA swizzle atoms need it)."""
    buf = torch.empty(nbytes + 1024, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % 1024
    return buf[off:off + nbytes]


def wino_conv2d(x, w, algo, pad=1, layout="nchw", out=None, workspace=None, stream=None):
    """y = conv(x, w) (valid cross-correlation, stride 1, zero padding `pad`)
    through libwino's kernels.  x: [N,C,H,W] ("nchw") or [N,H,W,C] ("nhwc"),
    w: [K,C,3,3], same dtype, same CUDA device; y in the layout of x.  Runs on
    `stream` (default: the current stream of x's device)."""
    if layout == "nchw":
        N, C, H, W = x.shape
    elif layout == "nhwc":
        N, H, W, C = x.shape
    else:
        raise WinoError(1, f"bad layout {layout!r}")
    K = w.shape[0]
    if not (x.is_cuda and w.is_cuda and x.device == w.device):
        raise WinoError(1, "x and w must be CUDA tensors on the same device")
    if tuple(w.shape) != (K, C, 3, 3) or w.dtype != x.dtype:
        raise WinoError(1, f"w must be [{K},{C},3,3] of dtype {x.dtype}; got {tuple(w.shape)} {w.dtype}")
    dt = _TORCH_DT.get(x.dtype)
    if dt is None:
        raise WinoError(1, f"unsupported dtype {x.dtype}")
    Ho, Wo = H + 2 * pad - 2, W + 2 * pad - 2
    shape = (N, K, Ho, Wo) if layout == "nchw" else (N, Ho, Wo, K)
    with torch.cuda.device(x.device):
        x = x.contiguous()
        w = w.contiguous()
        if out is None:
            out = torch.empty(shape, dtype=x.dtype, device=x.device)
        else:
            _check_out(out, shape, x.dtype, x.device)
        nbytes = wino_conv2d_workspace(algo, N, C, H, W, K, pad, dt, layout)
        if workspace is None:
            workspace = alloc_workspace(nbytes, x.device)
        elif workspace.device != x.device or workspace.numel() < nbytes:
            raise WinoError(6, f"workspace must hold {nbytes} bytes on {x.device}")
        _on_stream(stream, x, w, out, workspace)
        check(lib().wino_conv2d(_ptr(x), _ptr(w), N, C, H, W, K, pad, algo.handle, DTYPES[dt], LAYOUTS[layout],
                                _ptr(out), _ptr(workspace), workspace.numel(), _stream(stream, x.device)))
    return out


def wino_conv2d_host_io(x_host, x_dev, w, algo, out_dev, out_host, workspace, pad=1, stream=None, layout="nchw"):
    """End-to-end call: pinned host x -> device -> layer -> pinned host y, on `stream`."""
    if layout == "nchw":
        N, C, H, W = x_dev.shape
    else:
        N, H, W, C = x_dev.shape
    K = w.shape[0]
    dt = _TORCH_DT[x_dev.dtype]
    Ho, Wo = H + 2 * pad - 2, W + 2 * pad - 2
    shape = (N, K, Ho, Wo) if layout == "nchw" else (N, Ho, Wo, K)
    if x_host.is_cuda or out_host.is_cuda or not (x_host.is_pinned() and out_host.is_pinned()):
        raise WinoError(1, "x_host and out_host must be pinned host tensors")
    if x_host.numel() * x_host.element_size() != x_dev.numel() * x_dev.element_size() or not x_host.is_contiguous():
        raise WinoError(1, "x_host must be a contiguous host copy of x_dev's shape and dtype")
    if out_host.numel() * out_host.element_size() != out_dev.numel() * out_dev.element_size() \
            or not out_host.is_contiguous():
        raise WinoError(1, "out_host must be a contiguous host buffer of out_dev's size")
    _check_out(out_dev, shape, x_dev.dtype, x_dev.device)
    with torch.cuda.device(x_dev.device):
        _on_stream(stream, x_dev, w, out_dev, workspace)
        check(lib().wino_conv2d_host_io(_ptr(x_host), _ptr(x_dev), _ptr(w), N, C, H, W, K, pad, algo.handle,
                                        DTYPES[dt], LAYOUTS[layout], _ptr(out_dev), _ptr(out_host),
                                        _ptr(workspace), workspace.numel(), _stream(stream, x_dev.device)))


def geometry(algo, N, C, H, W, K, pad=1, dtype="bf16"):
    """Workspace geometry (mirrors include/wino.h): sizes of U, V, M."""
    m, D, S = algo.m, algo.domain, algo.units
    Ho, Wo = H + 2 * pad - 2, W + 2 * pad - 2
    th, tw = -(-Ho // m), -(-Wo // m)
    T = N * th * tw
    m16 = getattr(algo, "m_store", "fp32") == "dtype" and dtype != "fp32" and algo.m <= 8
    return dict(Ho=Ho, Wo=Wo, th=th, tw=tw, T=T, Tp=-(-T // 32) * 32, Cp=-(-C // 64) * 64, Q=D * D, S=S,
                planes=2 if dtype == "fp32" else 1, TB=-(-T // 128), CBW=32 if dtype == "fp32" else 64,
                mes=2 if m16 else 4)


def v_to_dense(V, T):
    """Blocked V [planes][TB][Cp/CBW][Q][128][CBW] (include/wino.h) -> dense
    [planes][Q][T][Cp] view for inspection (a copy)."""
    P_, TB, CB, Q, _, CBW = V.shape
    return V.permute(0, 3, 1, 4, 2, 5).reshape(P_, Q, TB * 128, CB * CBW)[:, :, :T]


def v_from_dense(Vd):
    """Dense [planes][Q][T][Cp] -> the blocked V layout the GEMM reads."""
    P_, Q, T, Cp = Vd.shape
    CBW = 32 if Vd.dtype == torch.float32 else 64
    TB = -(-T // 128)
    pad = torch.zeros((P_, Q, TB * 128, Cp), dtype=Vd.dtype, device=Vd.device)
    pad[:, :, :T] = Vd
    return pad.reshape(P_, Q, TB, 128, Cp // CBW, CBW).permute(0, 2, 4, 1, 3, 5).contiguous()


def wino_weight_transform(w, algo, stream=None):
    """U [planes][S][K][Cp] in the storage dtype (fp32: hi, lo planes)."""
    K, C = w.shape[:2]
    dt = _TORCH_DT[w.dtype]
    g = geometry(algo, 1, C, 3, 3, K, 1, dt)
    U = torch.empty((g["planes"], g["S"], K, g["Cp"]), dtype=w.dtype, device=w.device)
    with torch.cuda.device(w.device):
        check(lib().wino_weight_transform(_ptr(w.contiguous()), K, C, algo.handle, DTYPES[dt], _ptr(U),
                                          _stream(stream, w.device)))
    return U


def wino_input_transform(x, algo, pad=1, stream=None, layout="nchw"):
    """V [planes][TB][Cp/CBW][Q][128][CBW] (blocked, see v_to_dense) in the storage
    dtype; x [N,C,H,W] or [N,H,W,C] ("nhwc")."""
    if layout == "nchw":
        N, C, H, W = x.shape
    else:
        N, H, W, C = x.shape
    dt = _TORCH_DT[x.dtype]
    g = geometry(algo, N, C, H, W, 1, pad, dt)
    V = torch.empty((g["planes"], g["TB"], g["Cp"] // g["CBW"], g["Q"], 128, g["CBW"]), dtype=x.dtype,
                    device=x.device)
    with torch.cuda.device(x.device):
        check(lib().wino_input_transform(_ptr(x.contiguous()), N, C, H, W, pad, algo.handle, DTYPES[dt], LAYOUTS[layout],
                                         _ptr(V), _stream(stream, x.device)))
    return V


def wino_domain_gemm(V, U, algo, C, K, T, stream=None):
    """M [Q][K][Tp] from blocked V (T tiles) and U: fp32, or V's 16-bit dtype when
    the algorithm stores M in the dtype (set_m_storage, reading M3)."""
    dt = _TORCH_DT[V.dtype]
    Tp = -(-T // 32) * 32
    mdt = V.dtype if (algo.m_store == "dtype" and dt != "fp32" and algo.m <= 8) else torch.float32
    M = torch.empty((algo.domain ** 2, K, Tp), dtype=mdt, device=V.device)
    with torch.cuda.device(V.device):
        check(lib().wino_domain_gemm(_ptr(V), _ptr(U), T, C, K, algo.handle, DTYPES[dt], _ptr(M), _stream(stream, V.device)))
    return M


def wino_output_transform(M, algo, N, K, H, W, pad=1, dtype="bf16", stream=None, layout="nchw"):
    want = TORCH_OF[dtype] if (algo.m_store == "dtype" and dtype != "fp32" and algo.m <= 8) else torch.float32
    if M.dtype != want:
        raise WinoError(1, f"M must be {want} for this algorithm's M storage ({algo.m_store}); got {M.dtype}")
    Ho, Wo = H + 2 * pad - 2, W + 2 * pad - 2
    shape = (N, K, Ho, Wo) if layout == "nchw" else (N, Ho, Wo, K)
    y = torch.empty(shape, dtype=TORCH_OF[dtype], device=M.device)
    with torch.cuda.device(M.device):
        check(lib().wino_output_transform(_ptr(M), N, K, H, W, pad, algo.handle, DTYPES[dtype], LAYOUTS[layout],
                                          _ptr(y), _stream(stream, M.device)))
    return y


# --------------------------------------------------------------------------- 1D tiles / metrics


def wino_conv1d_tiles(x, h, algo, per_op_rounding=True, stream=None, bf16_mode="rne"):
    T = x.shape[0]
    assert x.shape == (T, algo.m + 2) and h.shape == (T, 3) and x.dtype == h.dtype
    y = torch.empty((T, algo.m), dtype=x.dtype, device=x.device)
    with torch.cuda.device(x.device):
        check(lib().wino_conv1d_tiles(_ptr(x.contiguous()), _ptr(h.contiguous()), T, algo.handle, _dt(x),
                                      (1 if per_op_rounding else 0) | (2 if bf16_mode == "trunc" else 0), _ptr(y),
                                      _stream(stream, x.device)))
    return y


def wino_conv2d_tiles_paper(d, g, algo, csum="sequential", acc="dtype", bf16_mode="rne", stream=None):
    """Paper-mode multi-channel 2D tiles: d [C][S][m+2][m+2], g [C][S][3][3] ->
    Y [S][m][m] (include/wino.h wino_conv2d_tiles_paper)."""
    C, S = d.shape[:2]
    nx = algo.m + 2
    if tuple(d.shape) != (C, S, nx, nx) or tuple(g.shape) != (C, S, 3, 3) or d.dtype != g.dtype:
        raise WinoError(1, "d must be [C][S][m+2][m+2] and g [C][S][3][3] of one dtype")
    y = torch.empty((S, algo.m, algo.m), dtype=d.dtype, device=d.device)
    with torch.cuda.device(d.device):
        check(lib().wino_conv2d_tiles_paper(_ptr(d.contiguous()), _ptr(g.contiguous()), C, S, algo.handle, _dt(d),
                                            {"sequential": 0, "pairwise": 1}[csum], {"dtype": 0, "fp32": 1}[acc],
                                            {"rne": 0, "trunc": 1}[bf16_mode], _ptr(y), _stream(stream, d.device)))
    return y


def wino_error_stats(y, y_ref, m, stream=None):
    """8 fp64 statistics (include/wino.h) of y vs the fp64 reference, on the device."""
    N, K, Ho, Wo = y.shape
    assert y_ref.shape == y.shape and y_ref.dtype == torch.float64
    stats = torch.empty(8, dtype=torch.float64, device=y.device)
    nbytes = lib().wino_error_stats_scratch(N, K, Ho, Wo, m)
    scratch = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=y.device)
    with torch.cuda.device(y.device):
        check(lib().wino_error_stats(_ptr(y.contiguous()), _dt(y), _ptr(y_ref.contiguous()), N, K, Ho, Wo, m,
                                     _ptr(stats), _ptr(scratch), _stream(stream, y.device)))
    return stats


def wino_direct_conv2d_f64(x, w, pad=1, stream=None):
    N, C, H, W = x.shape
    K = w.shape[0]
    y = torch.empty((N, K, H + 2 * pad - 2, W + 2 * pad - 2), dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        check(lib().wino_direct_conv2d_f64(_ptr(x.contiguous()), _ptr(w.contiguous()), N, C, H, W, K, pad, _dt(x),
                                           _ptr(y), _stream(stream, x.device)))
    return y


def wino_last_launch_count():
    return int(lib().wino_last_launch_count())


def summary(stats):
    s = stats.tolist() if hasattr(stats, "tolist") else list(stats)
    return {"rel_l1": s[0] / s[1] if s[1] else float("nan"), "mean_rel": s[2] / s[6],
            "mean_euclid": s[3] / s[6], "max_rel": s[4], "nonfinite": int(s[5]), "tiles": int(s[6])}
