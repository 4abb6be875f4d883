"""Emulated floating point (oracle component O9).  Test infrastructure only.

Rounding primitives (readings A10, A11 in DESIGN.md): round-to-nearest-even
everywhere, subnormals kept, overflow to +-inf.  bf16 "a truncated form of fp32"
(P:6) is read as the *format*; a truncation mode is available as a switch.

Two precision models of the 2D layer / 1D tiles:

PAPER mode ("performing the operations in single precision and casting
  the results to the lower precision"): every scalar multiply and add is done in
  fp32 and its result is cast to the dtype; dot products accumulate in ascending
  index order, starting from the first product; matrix entries are rounded once
  to the dtype.  Zero matrix entries are multiplied like any other (dense
  evaluation).

PIPELINE mode (the rounding points of the staged GPU path): x and w are dtype
  values; U = rd(G g G^T), V = rd(B^T d B) computed in fp32 with fp32-lowered
  matrices; M = sum_c U V accumulated in fp32; y = rd(A^T M A) computed in fp32.
  The order of fp32 operations inside each stage is not part of the model.
  m_store="dtype" (reading M3, the layer form of the "mixed
  precision" booster of P:611 / reading M2): the fp32 channel sum M is rounded
  once to the dtype before the output transform, y = rd(A^T rd(M) A).

The absolute error magnitudes these models produce are "parity unpinned"
(Figure 1 is absent from PAPER.md); their trends are pinned in tests.
"""
from fractions import Fraction
import numpy as np

from . import conv as CV

UNIT_ROUNDOFF = {"fp32": 2.0 ** -24, "fp16": 2.0 ** -11, "bf16": 2.0 ** -8, "fp64": 2.0 ** -53}


# --------------------------------------------------------------------------- rounding primitives


def frac_to_f32(fr):
    """Correctly rounded (RNE) fp32 of an exact rational (the fp32 lowering of a
    transform-matrix entry)."""
    fr = Fraction(fr)
    f = np.float32(float(fr))
    best, best_err = None, None
    for c in (np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))):
        err = abs(Fraction(float(c)) - fr)
        if best is None or err < best_err or (err == best_err and (int(np.float32(c).view(np.uint32)) & 1) == 0):
            best, best_err = np.float32(c), err
    return best


def lower_f32(mat):
    return np.array([[frac_to_f32(v) for v in row] for row in mat], dtype=np.float32)


def rd_fp32(a):
    return np.asarray(a).astype(np.float32)


def rd_fp16(a32):
    """fp32 -> fp16 (RNE, subnormals, overflow -> inf), returned as fp32 values."""
    a32 = np.asarray(a32, dtype=np.float32)
    with np.errstate(over="ignore"):
        return a32.astype(np.float16).astype(np.float32)


def rd_bf16(a32, mode="rne"):
    """fp32 -> bf16 by bit manipulation of the fp32 pattern, returned as fp32
    values.  mode 'rne' rounds to nearest even; mode 'trunc' drops the low 16
    bits."""
    a32 = np.ascontiguousarray(np.asarray(a32, dtype=np.float32))
    bits = a32.view(np.uint32).astype(np.uint64)
    if mode == "trunc":
        r = bits & 0xFFFF0000
    else:
        r = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    nan = np.isnan(a32)
    r = np.where(nan, (bits & 0xFFFF0000) | 0x00400000, r)
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def rd(dtype, a32, bf16_mode="rne"):
    if dtype == "fp32":
        return rd_fp32(a32)
    if dtype == "fp16":
        return rd_fp16(a32)
    if dtype == "bf16":
        return rd_bf16(a32, bf16_mode)
    if dtype == "fp64":
        return np.asarray(a32, np.float64)
    raise ValueError(dtype)


# --------------------------------------------------------------------------- separable helpers


def sep2(Mat, arr):
    """out[p, q, ...] = sum_{a, b} Mat[p, a] Mat[q, b] arr[a, b, ...] in the dtype of
    the operands (fp32 here: two library GEMM stages, rows then columns)."""
    a, b = arr.shape[:2]
    rest = arr.shape[2:]
    R = int(np.prod(rest)) if rest else 1
    t1 = (Mat @ arr.reshape(a, b * R)).reshape(Mat.shape[0], b, R)
    t2 = np.matmul(Mat, t1)                                  # (p, q, R)
    return t2.reshape((Mat.shape[0], Mat.shape[0]) + rest)


def halo_tiles(x, m, nx, pad):
    """x[N, C, H, W] -> d[nx, nx, N, C, th, tw]: d[a, b, n, c, ti, tj] =
    x[n, c, ti*m - pad + a, tj*m - pad + b], zero outside."""
    N, C, H, W = x.shape
    Ho, Wo, th, tw = CV.tile_grid(H, W, m, pad, nx - m + 1)
    xp = np.zeros((N, C, th * m + nx - m, tw * m + nx - m), x.dtype)
    hh, ww = min(H, xp.shape[2] - pad), min(W, xp.shape[3] - pad)
    xp[:, :, pad:pad + hh, pad:pad + ww] = x[:, :, :hh, :ww]
    d = np.empty((nx, nx, N, C, th, tw), x.dtype)
    for a in range(nx):
        for b in range(nx):
            d[a, b] = xp[:, :, a:a + m * th:m, b:b + m * tw:m]
    return d, (Ho, Wo, th, tw)


def _scatter_tiles(Yt, N, K, th, tw, m, Ho, Wo):
    """Yt[p, q, K, N*th*tw] -> y[N, K, Ho, Wo] (outputs beyond Ho, Wo discarded)."""
    Y = Yt.reshape(m, m, K, N, th, tw).transpose(3, 2, 4, 0, 5, 1).reshape(N, K, th * m, tw * m)
    return Y[:, :, :Ho, :Wo]


# --------------------------------------------------------------------------- pipeline mode, 2D layer


def pipeline_weight_transform(ts, w, dtype, bf16_mode="rne"):
    """U[i, j, k, c] = rd((G g_{k,c} G^T)_{ij}) in fp32 (Eq. 2 'G H G^T')."""
    G = lower_f32(ts.G)
    w32 = np.asarray(w, np.float32).transpose(2, 3, 0, 1)            # (3, 3, K, C)
    return rd(dtype, sep2(G, w32), bf16_mode)


def pipeline_input_transform(ts, x, dtype, pad=1, bf16_mode="rne"):
    """V[i, j, t, c] = rd((B^T d_{t,c} B)_{ij}) in fp32 (Eq. 2 'B^T X B'); t =
    (n, ti, tj) row-major."""
    BT = lower_f32(ts.BT)
    d, grid = halo_tiles(np.asarray(x, np.float32), ts.n_o, ts.n_x, pad)
    V = rd(dtype, sep2(BT, d), bf16_mode)                            # (mu, mu, N, C, th, tw)
    mu = ts.mu
    N, C = d.shape[2], d.shape[3]
    V = V.transpose(0, 1, 2, 4, 5, 3).reshape(mu, mu, -1, C)         # (mu, mu, T, C)
    return V, grid


def pipeline_conv2d(ts, x, w, dtype, pad=1, bf16_mode="rne", chunk=16, return_parts=False, m_store="fp32"):
    """Whole layer in PIPELINE mode.  x: [N, C, H, W] dtype values (any float
    array), w: [K, C, 3, 3].  Returns y as fp32 array of dtype values.
    m_store: "fp32" (reading R1) or "dtype" (reading M3: M rounded once)."""
    assert m_store in ("fp32", "dtype")
    x = np.asarray(x)
    N, C, H, W = x.shape
    K = w.shape[0]
    m, mu = ts.n_o, ts.mu
    U = pipeline_weight_transform(ts, w, dtype, bf16_mode)             # (mu, mu, K, C)
    AT = lower_f32(ts.AT)
    Ho, Wo, th, tw = CV.tile_grid(H, W, m, pad, ts.n_h)
    y = np.empty((N, K, Ho, Wo), np.float32)
    parts = {"U": U, "V": [], "M": []}
    for n0 in range(0, N, chunk):
        xs = x[n0:n0 + chunk]
        V, _ = pipeline_input_transform(ts, xs, dtype, pad, bf16_mode)
        Mx = np.matmul(U, V.transpose(0, 1, 3, 2))                   # (mu, mu, K, T) fp32 accumulate
        if m_store == "dtype":
            with np.errstate(over="ignore"):
                Mx = rd(dtype, Mx, bf16_mode)                        # M3: one rounding of the channel sum
        Yt = rd(dtype, sep2(AT, Mx), bf16_mode)                      # (m, m, K, T)
        y[n0:n0 + chunk] = _scatter_tiles(Yt, xs.shape[0], K, th, tw, m, Ho, Wo)
        if return_parts:
            parts["V"].append(V)
            parts["M"].append(Mx)
    if return_parts:
        return y, parts
    return y


# --------------------------------------------------------------------------- pipeline mode, residue lowering


def residue_slabs(rb):
    """Enumerate the GEMM units of the residue-block lowering (O6).  Returns a
    list of (out_point, in_point, kr, kc) where out/in points index the D x D
    domain row-major, and the unit's weight is
        W = sum_{a in I, b in J} U[a, b] * Phi_a[k'_loc, k_loc] * Phi_b[l'_loc, l_loc]."""
    units = []
    D = rb.D
    for (sI, nI, _), phI in zip(rb.blocks, rb.phi):
        for (sJ, nJ, _), phJ in zip(rb.blocks, rb.phi):
            for k in range(nI):
                for l in range(nJ):
                    for kk in range(nI):
                        for ll in range(nJ):
                            units.append(((sI + k) * D + (sJ + l), (sI + kk) * D + (sJ + ll),
                                          (sI, nI, phI), (sJ, nJ, phJ), (k, l, kk, ll)))
    return units


def pipeline_residue_weights(rb, w, dtype, bf16_mode="rne"):
    """W_unit[k, c] = rd(sum_{a, b} U[a, b] Phi_a[kk, k] Phi_b[ll, l]) with the
    unrounded fp32 U = G_P g G_P^T; the combination is formed in fp32, ascending
    (a, b), and rounded once."""
    GP = lower_f32(rb.GP)
    w32 = np.asarray(w, np.float32).transpose(2, 3, 0, 1)
    U = sep2(GP, w32)                                                  # (D, D, K, C) fp32, unrounded
    units = residue_slabs(rb)
    Ws = []
    for (_, _, (sI, nI, phI), (sJ, nJ, phJ), (k, l, kk, ll)) in units:
        acc = None
        for a in range(nI):
            for b in range(nJ):
                coef = phI[a][kk][k] * phJ[b][ll][l]
                if coef == 0:
                    continue
                term = np.float32(frac_to_f32(coef)) * U[sI + a, sJ + b]
                acc = term if acc is None else (acc + term).astype(np.float32)
        if acc is None:
            acc = np.zeros_like(U[0, 0])
        Ws.append(rd(dtype, acc, bf16_mode))
    return units, np.stack(Ws)                                        # (n_units, K, C)


def pipeline_residue_conv2d(rb, x, w, dtype, pad=1, bf16_mode="rne", chunk=16, m_store="fp32"):
    assert m_store in ("fp32", "dtype")
    x = np.asarray(x)
    N, C, H, W = x.shape
    K = w.shape[0]
    m, D = rb.n_o, rb.D
    nx = m + rb.n_h - 1
    units, Wst = pipeline_residue_weights(rb, w, dtype, bf16_mode)
    BPT = lower_f32([list(r) for r in zip(*rb.BP)])                  # D x nx
    APT = lower_f32([list(r) for r in zip(*rb.AP)])                  # m x D
    Ho, Wo, th, tw = CV.tile_grid(H, W, m, pad, rb.n_h)
    y = np.empty((N, K, Ho, Wo), np.float32)
    for n0 in range(0, N, chunk):
        xs = np.asarray(x[n0:n0 + chunk], np.float32)
        d, _ = halo_tiles(xs, m, nx, pad)
        V = rd(dtype, sep2(BPT, d), bf16_mode)                        # (D, D, n, C, th, tw)
        V = V.transpose(0, 1, 2, 4, 5, 3).reshape(D * D, -1, C)       # (D^2, T, C)
        Z = np.zeros((D * D, K, V.shape[1]), np.float32)
        for u, (po, pi, *_rest) in enumerate(units):
            Z[po] = (Z[po] + Wst[u] @ V[pi].T).astype(np.float32)
        if m_store == "dtype":
            with np.errstate(over="ignore"):
                Z = rd(dtype, Z, bf16_mode)                          # M3: one rounding of the domain sum
        Yt = rd(dtype, sep2(APT, Z.reshape(D, D, K, -1)), bf16_mode)
        y[n0:n0 + chunk] = _scatter_tiles(Yt, xs.shape[0], K, th, tw, m, Ho, Wo)
    return y


# --------------------------------------------------------------------------- paper mode (per scalar op)


def po_matmul(Mat, X, dtype, bf16_mode="rne"):
    """out[i, ...] = sum_j Mat[i, j] X[j, ...] with every product and every
    partial sum computed in fp32 and cast to the dtype, ascending j, starting
    from the first product."""
    Mat = np.asarray(Mat, np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        return _po_matmul(Mat, X, dtype, bf16_mode)


def _po_matmul(Mat, X, dtype, bf16_mode):
    out = []
    for i in range(Mat.shape[0]):
        acc = rd(dtype, Mat[i, 0] * X[0], bf16_mode)
        for j in range(1, Mat.shape[1]):
            p = rd(dtype, Mat[i, j] * X[j], bf16_mode)
            acc = rd(dtype, (acc + p).astype(np.float32), bf16_mode)
        out.append(acc)
    return np.stack(out)


def paper_matrices(ts, dtype, bf16_mode="rne"):
    """Matrix entries rounded once to the dtype."""
    return (rd(dtype, lower_f32(ts.G), bf16_mode), rd(dtype, lower_f32(ts.BT), bf16_mode),
            rd(dtype, lower_f32(ts.AT), bf16_mode))


def paper_conv1d(ts, x, h, dtype, bf16_mode="rne"):
    """Batched 1D tiles in PAPER mode (BASELINE cfg 2): x[T, n_x], h[T, 3] ->
    y[T, n_o]; u = G h, v = B^T x, p = u (.) v, y = A^T p, each op per P:556."""
    G, BT, AT = paper_matrices(ts, dtype, bf16_mode)
    xt = np.asarray(x, np.float32).T
    ht = np.asarray(h, np.float32).T
    u = po_matmul(G, ht, dtype, bf16_mode)
    v = po_matmul(BT, xt, dtype, bf16_mode)
    p = rd(dtype, (u * v).astype(np.float32), bf16_mode)
    return po_matmul(AT, p, dtype, bf16_mode).T


def pipeline_conv1d(ts, x, h, dtype, bf16_mode="rne"):
    """Batched 1D tiles in PIPELINE mode: u = rd(G h), v = rd(B^T x) in fp32,
    p = u v in fp32, y = rd(A^T p) in fp32."""
    G, BT, AT = lower_f32(ts.G), lower_f32(ts.BT), lower_f32(ts.AT)
    u = rd(dtype, G @ np.asarray(h, np.float32).T, bf16_mode)
    v = rd(dtype, BT @ np.asarray(x, np.float32).T, bf16_mode)
    p = (u * v).astype(np.float32)
    return rd(dtype, AT @ p, bf16_mode).T


def pairwise_sum(terms, add):
    """Pairwise (tree) summation over channels, one of the accuracy boosters
    P:611 lists as composable with the method ("pairwise summation over
    channels"): sum(t[0:n]) = add(sum(t[0:h]), sum(t[h:n])) with h the largest
    power of two below n -- the same tree as combining adjacent pairs level by
    level and carrying an odd last element up unchanged."""
    n = len(terms)
    if n == 1:
        return terms[0]
    h = 1
    while 2 * h < n:
        h *= 2
    return add(pairwise_sum(terms[:h], add), pairwise_sum(terms[h:], add))


def paper_conv2d_tiles(ts, d, g, dtype, bf16_mode="rne", csum="sequential", acc="dtype"):
    """PAPER mode on a batch of single-channel-summed tile samples:
    d[C, S, n_x, n_x], g[C, S, 3, 3] -> Y[S, m, m].  Kernel transform rows then
    columns, input transform rows then columns, product, channel sum in the
    Winograd domain, output transform rows then columns; every op per P:556.

    Channel sum variants (composable accuracy boosters; readings M1, M2 in
    DESIGN.md): csum = "sequential" (ascending c, the paper's baseline) or
    "pairwise" (pairwise_sum); acc = "dtype" (every partial sum cast to the
    dtype) or "fp32" (mixed precision: the rounded products P_c are accumulated
    in fp32 and the channel sum is cast to the dtype once, before the output
    transform)."""
    G, BT, AT = paper_matrices(ts, dtype, bf16_mode)
    d = np.asarray(d, np.float32)
    g = np.asarray(g, np.float32)
    prods = []
    for c in range(d.shape[0]):
        gc = g[c].transpose(1, 2, 0)                                  # (3, 3, S)
        dc = d[c].transpose(1, 2, 0)                                  # (nx, nx, S)
        U = po_matmul(G, gc, dtype, bf16_mode)                        # (mu, 3, S)
        U = po_matmul(G, U.transpose(1, 0, 2), dtype, bf16_mode).transpose(1, 0, 2)
        V = po_matmul(BT, dc, dtype, bf16_mode)
        V = po_matmul(BT, V.transpose(1, 0, 2), dtype, bf16_mode).transpose(1, 0, 2)
        with np.errstate(over="ignore", invalid="ignore"):
            prods.append(rd(dtype, (U * V).astype(np.float32), bf16_mode))
    if acc == "dtype":
        def add(a, b):
            with np.errstate(over="ignore", invalid="ignore"):
                return rd(dtype, (a + b).astype(np.float32), bf16_mode)
    elif acc == "fp32":
        def add(a, b):
            with np.errstate(over="ignore", invalid="ignore"):
                return (a + b).astype(np.float32)
    else:
        raise ValueError(acc)
    if csum == "sequential":
        Msum = prods[0]
        for P_c in prods[1:]:
            Msum = add(Msum, P_c)
    elif csum == "pairwise":
        Msum = pairwise_sum(prods, add)
    else:
        raise ValueError(csum)
    if acc == "fp32":
        with np.errstate(over="ignore"):
            Msum = rd(dtype, Msum, bf16_mode)
    Y = po_matmul(AT, Msum, dtype, bf16_mode)
    Y = po_matmul(AT, Y.transpose(1, 0, 2), dtype, bf16_mode).transpose(1, 0, 2)
    return Y.transpose(2, 0, 1)


# --------------------------------------------------------------------------- forward error bound


def abs_bound_conv2d(ts, x, w, dtype, pad=1, C_acc=None, mma_rel=0.0):
    """First-order running-error analysis of the pipeline model (DESIGN.md
    "Parity bounds"); see elementwise_bound for the complete bound.  Returns
    (S, g, u_d):  S = |A|^T ( sum_c (|G||g||G|^T) (.) (|B|^T|d||B|) ) |A|,
    g = (8 + 2 n_x + 2 + C + 2 mu + 2) u_32 + mma_rel."""
    S, g, u_d, _ = _abs_bound_parts(ts, x, w, dtype, pad, C_acc, mma_rel)
    return S, g, u_d


# half the smallest subnormal: the absolute error of rounding an underflowing value
ETA = {"fp32": 2.0 ** -150, "fp16": 2.0 ** -25, "bf16": 2.0 ** -134, "fp64": 0.0}


def elementwise_bound(ts, x, w, dtype, yref, pad=1, mma_rel=0.0, safety=1.05, m_store="fp32"):
    """|y_pipeline - y_exact| <= (2 u_d + g) S + eta S_eta + u_d |y| + eta, with
    S_eta = |A|^T ( sum_c (|G||g||G|^T) + (|B|^T|d||B|) + eta ) |A| the
    propagation of underflow (absolute) errors of U and V (fp16 lin8 collapse).
    m_store="dtype" (reading M3) adds the rounding of M, |rd(M) - M| <= u_d |M|
    + eta, propagated by |A|^T . |A|: + u_d S + eta (max_p sum_i |A_ip|)^2."""
    S, g, u_d, S_eta = _abs_bound_parts(ts, x, w, dtype, pad, None, mma_rel)
    eta = ETA[dtype]
    b = (2 * u_d + g) * S + eta * S_eta + u_d * np.abs(yref) + eta
    if m_store == "dtype":
        a1 = np.abs(np.array([[float(v) for v in r] for r in ts.AT])).sum(axis=1).max()
        b = b + u_d * S + eta * a1 * a1
    return safety * b


def _abs_bound_parts(ts, x, w, dtype, pad, C_acc, mma_rel):
    u_d = UNIT_ROUNDOFF[dtype]
    u32 = UNIT_ROUNDOFF["fp32"]
    C = x.shape[1]
    C_acc = C if C_acc is None else C_acc
    absG = np.abs(np.array([[float(v) for v in r] for r in ts.G]))
    absBT = np.abs(np.array([[float(v) for v in r] for r in ts.BT]))
    absAT = np.abs(np.array([[float(v) for v in r] for r in ts.AT]))
    m, mu = ts.n_o, ts.mu
    N, _, H, W = x.shape
    K = w.shape[0]
    Ua = sep2(absG, np.abs(np.asarray(w, np.float64)).transpose(2, 3, 0, 1))          # (mu, mu, K, C)
    d, (Ho, Wo, th, tw) = halo_tiles(np.abs(np.asarray(x, np.float64)), m, ts.n_x, pad)
    Va = sep2(absBT, d).transpose(0, 1, 2, 4, 5, 3).reshape(mu, mu, -1, C)            # (mu, mu, T, C)
    Ma = np.matmul(Ua, Va.transpose(0, 1, 3, 2))
    S = _scatter_tiles(sep2(absAT, Ma), N, K, th, tw, m, Ho, Wo)
    eta = ETA[dtype]
    Me = Ua.sum(axis=3)[:, :, :, None] + Va.sum(axis=3)[:, :, None, :] + eta * C        # (mu, mu, K, T)
    S_eta = _scatter_tiles(sep2(absAT, Me), N, K, th, tw, m, Ho, Wo)
    g = (8 + 2 * ts.n_x + 2 + C_acc + 2 * mu + 2) * u32 + mma_rel
    return S, g, u_d, S_eta


def residue_elementwise_bound(rb, x, w, dtype, yref, pad=1, mma_rel=0.0, safety=1.05, m_store="fp32"):
    """First-order forward error bound of the residue-block pipeline
    (pipeline_residue_conv2d; reading R1 applied to A3'):
        |y - y_exact| <= (2 u_d + g) S + eta S_eta + u_d |y| + eta,
    with S = |A_P|^T ( sum_units sum_c |W_unit| |V_in| ) |A_P| scattered to the
    outputs, |W_unit| <= sum_terms |coef| (|G_P| |g| |G_P|^T)_term (the slab
    combination before its single rounding), |V| <= |B_P|^T |d| |B_P|, and g the
    fp32 error of the transforms, the slab combination (<= 4 terms) and the
    channel x unit accumulation of each output point.  S_eta propagates the
    absolute (underflow) errors of W and V."""
    u_d = UNIT_ROUNDOFF[dtype]
    u32 = UNIT_ROUNDOFF["fp32"]
    m, D, nh = rb.n_o, rb.D, rb.n_h
    nx = m + nh - 1
    C = x.shape[1]
    N, _, H, W = x.shape
    K = w.shape[0]
    absGP = np.abs(np.array([[float(v) for v in r] for r in rb.GP]))
    absBPT = np.abs(np.array([[float(v) for v in r] for r in zip(*rb.BP)]))      # D x nx
    absAPT = np.abs(np.array([[float(v) for v in r] for r in zip(*rb.AP)]))      # m x D
    Ua = sep2(absGP, np.abs(np.asarray(w, np.float64)).transpose(2, 3, 0, 1))    # (D, D, K, C)
    d, (Ho, Wo, th, tw) = halo_tiles(np.abs(np.asarray(x, np.float64)), m, nx, pad)
    Va = sep2(absBPT, d).transpose(0, 1, 2, 4, 5, 3).reshape(D * D, -1, C)        # (D^2, T, C)
    Tn = Va.shape[1]
    Z = np.zeros((D * D, K, Tn))
    Ze = np.zeros((D * D, K, Tn))
    per_point = np.zeros(D * D, int)
    eta = ETA[dtype]
    for (po, pi, (sI, nI, phI), (sJ, nJ, phJ), (k, l, kk, ll)) in residue_slabs(rb):
        Wa = np.zeros((K, C))
        for a in range(nI):
            for b in range(nJ):
                coef = abs(float(phI[a][kk][k] * phJ[b][ll][l]))
                if coef:
                    Wa += coef * Ua[sI + a, sJ + b]
        Z[po] += Wa @ Va[pi].T
        Ze[po] += Wa.sum(axis=1)[:, None] + Va[pi].sum(axis=1)[None, :] + eta * C
        per_point[po] += 1
    S = _scatter_tiles(sep2(absAPT, Z.reshape(D, D, K, Tn)), N, K, th, tw, m, Ho, Wo)
    S_eta = _scatter_tiles(sep2(absAPT, Ze.reshape(D, D, K, Tn)), N, K, th, tw, m, Ho, Wo)
    g = (8 + 2 * nx + 2 + 4 + C * int(per_point.max()) + 2 * D + 2) * u32 + mma_rel
    b = (2 * u_d + g) * S + eta * S_eta + u_d * np.abs(yref) + eta
    if m_store == "dtype":   # reading M3: the domain sum rounded once (see elementwise_bound)
        b = b + u_d * S + eta * absAPT.sum(axis=1).max() ** 2
    return safety * b
