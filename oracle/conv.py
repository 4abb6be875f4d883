"""Direct and exact-Winograd convolution (oracle components O5, O7, O8).
Test infrastructure only.

* Direct convolution in the DNN sense: valid cross-correlation, no kernel flip
  (reading A5; "the simple direct algorithm"), stride 1, zero padding.
* Exact Winograd, Eq. (2): Y = A^T [(G g G^T) (.) (B^T d B)] A, with
  the role assignment of reading A4 (see transforms.TransformSet).
* Tiling: overlapping n_x x n_x input tiles at stride n_o, halo origin
  (t_i*m - pad, t_j*m - pad), zeros outside the image, ragged edges discarded
  (reading A18); the channel sum is taken in the Winograd domain.
"""
from fractions import Fraction
import numpy as np


def tile_grid(H, W, m, pad, r=3):
    """Output size and tile counts for stride 1: H_out = H + 2 pad - r + 1."""
    Ho, Wo = H + 2 * pad - r + 1, W + 2 * pad - r + 1
    return Ho, Wo, -(-Ho // m), -(-Wo // m)


# --------------------------------------------------------------------------- direct


def direct_corr_1d(h, x):
    """y_j = sum_k h_k x_{j+k} (valid correlation), ascending k."""
    n = len(x) - len(h) + 1
    return [sum((h[k] * x[j + k] for k in range(len(h))), type(h[0])(0)) for j in range(n)]


def direct_corr_2d(g, d):
    r = len(g)
    n = len(d) - r + 1
    return [[sum((g[p][q] * d[i + p][j + q] for p in range(r) for q in range(r)), type(g[0][0])(0))
             for j in range(n)] for i in range(n)]


def direct_conv2d_f64(x, w, pad=1):
    """fp64 direct convolution of a layer (O7): x[N,C,H,W], w[K,C,3,3] ->
    y[N,K,Ho,Wo].  Summed over taps (p, q) in ascending order, each tap one
    library contraction over channels (a BLAS GEMM)."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    N, C, H, Wd = x.shape
    K, C2, r, r2 = w.shape
    assert C == C2 and r == r2
    Ho, Wo = H + 2 * pad - r + 1, Wd + 2 * pad - r + 1
    xp = np.zeros((N, C, H + 2 * pad, Wd + 2 * pad), np.float64)
    xp[:, :, pad:pad + H, pad:pad + Wd] = x
    y = np.zeros((N, K, Ho, Wo), np.float64)
    for p in range(r):
        for q in range(r):
            win = xp[:, :, p:p + Ho, q:q + Wo]                       # N C Ho Wo
            y += np.einsum("kc,nchw->nkhw", w[:, :, p, q], win, optimize=True)
    return y


def direct_conv2d_exact(x, w, pad=1):
    """Exact (object/Fraction) direct convolution, brute force, for tiny inputs."""
    N, C, H, Wd = len(x), len(x[0]), len(x[0][0]), len(x[0][0][0])
    K, r = len(w), len(w[0][0])
    Ho, Wo = H + 2 * pad - r + 1, Wd + 2 * pad - r + 1

    def px(n, c, i, j):
        i, j = i - pad, j - pad
        return x[n][c][i][j] if 0 <= i < H and 0 <= j < Wd else Fraction(0)

    return [[[[sum((w[k][c][p][q] * px(n, c, i + p, j + q)
                    for c in range(C) for p in range(r) for q in range(r)), Fraction(0))
               for j in range(Wo)] for i in range(Ho)] for k in range(K)] for n in range(N)]


# --------------------------------------------------------------------------- exact Winograd


def _mv(M, v):
    return [sum((M[i][j] * v[j] for j in range(len(v))), Fraction(0)) for i in range(len(M))]


def _mm(P, Q):
    return [[sum((P[i][t] * Q[t][j] for t in range(len(Q))), Fraction(0)) for j in range(len(Q[0]))]
            for i in range(len(P))]


def _tr(P):
    return [list(r) for r in zip(*P)]


def winograd_1d_exact(ts, h, x):
    """y = A^T [(G h) (.) (B^T x)] (P:92 Hadamard product; matrix exchange of P:94)."""
    u = _mv(ts.G, h)
    v = _mv(ts.BT, x)
    return _mv(ts.AT, [a * b for a, b in zip(u, v)])


def winograd_2d_exact(ts, g, d):
    """Eq. (2): A^T [(G g G^T) (.) (B^T d B)] A, one tile."""
    U = _mm(_mm(ts.G, g), _tr(ts.G))
    V = _mm(_mm(ts.BT, d), ts.B)
    P = [[U[i][j] * V[i][j] for j in range(len(U))] for i in range(len(U))]
    return _mm(_mm(ts.AT, P), ts.A)


def halo_tile(x_nc, ti, tj, m, nx, pad):
    """n_x x n_x input tile at origin (ti*m - pad, tj*m - pad), zero outside."""
    H, Wd = len(x_nc), len(x_nc[0])
    out = []
    for a in range(nx):
        row = []
        for b in range(nx):
            i, j = ti * m - pad + a, tj * m - pad + b
            row.append(x_nc[i][j] if 0 <= i < H and 0 <= j < Wd else Fraction(0))
        out.append(row)
    return out


def tiled_winograd_exact(ts, x, w, pad=1):
    """Exact tiled multi-channel layer (O8): per tile, sum over channels of
    (G g G^T) (.) (B^T d B) in the Winograd domain, one output transform per
    tile, ragged outputs discarded."""
    N, C, H, Wd = len(x), len(x[0]), len(x[0][0]), len(x[0][0][0])
    K = len(w)
    m, nx, u = ts.n_o, ts.n_x, ts.mu
    Ho, Wo, th, tw = tile_grid(H, Wd, m, pad, ts.n_h)
    Us = [[_mm(_mm(ts.G, w[k][c]), _tr(ts.G)) for c in range(C)] for k in range(K)]
    y = [[[[None] * Wo for _ in range(Ho)] for _ in range(K)] for _ in range(N)]
    for n in range(N):
        for ti in range(th):
            for tj in range(tw):
                Vs = [_mm(_mm(ts.BT, halo_tile(x[n][c], ti, tj, m, nx, pad)), ts.B) for c in range(C)]
                for k in range(K):
                    Mx = [[sum((Us[k][c][i][j] * Vs[c][i][j] for c in range(C)), Fraction(0))
                           for j in range(u)] for i in range(u)]
                    Y = _mm(_mm(ts.AT, Mx), ts.A)
                    for a in range(m):
                        for b in range(m):
                            i, j = ti * m + a, tj * m + b
                            if i < Ho and j < Wo:
                                y[n][k][i][j] = Y[a][b]
    return y


# --------------------------------------------------------------------------- residue-block lowering (exact)


def residue_1d_exact(rb, h, x):
    """y = A_P^T blockdiag(Phi(u_i)^T) B_P^T x with u = G_P h (transforms.ResidueBlocks)."""
    from .transforms import residue_weight_1d
    u = _mv(rb.GP, h)
    v = _mv(_tr(rb.BP), x)
    z = _mv(residue_weight_1d(rb, u), v)
    return _mv(_tr(rb.AP), z)


def residue_2d_exact(rb, g, d):
    """2D residue lowering, one tile: U = G_P g G_P^T, V = B_P^T d B_P, and for
    every block pair (I, J): Z_IJ = sum_{a in I, b in J} U[a, b] Phi_a^T V_IJ Phi_b;
    Y = A_P^T Z A_P."""
    U = _mm(_mm(rb.GP, g), _tr(rb.GP))
    V = _mm(_mm(_tr(rb.BP), d), rb.BP)
    Z = residue_bilinear_2d(rb, U, V)
    return _mm(_mm(_tr(rb.AP), Z), rb.AP)


def residue_bilinear_2d(rb, U, V):
    D = rb.D
    Z = [[Fraction(0)] * D for _ in range(D)]
    for (sI, nI, _), phI in zip(rb.blocks, rb.phi):
        for (sJ, nJ, _), phJ in zip(rb.blocks, rb.phi):
            for a in range(nI):
                for b in range(nJ):
                    uab = U[sI + a][sJ + b]
                    # Phi_a^T V_IJ Phi_b
                    for k in range(nI):
                        for l in range(nJ):
                            acc = Fraction(0)
                            for kk in range(nI):
                                for ll in range(nJ):
                                    acc += phI[a][kk][k] * V[sI + kk][sJ + ll] * phJ[b][ll][l]
                            Z[sI + k][sJ + l] += uab * acc
    return Z


def tiled_residue_exact(rb, x, w, pad=1):
    N, C, H, Wd = len(x), len(x[0]), len(x[0][0]), len(x[0][0][0])
    K = len(w)
    m, nx = rb.n_o, rb.n_o + rb.n_h - 1
    Ho, Wo, th, tw = tile_grid(H, Wd, m, pad, rb.n_h)
    Us = [[_mm(_mm(rb.GP, w[k][c]), _tr(rb.GP)) for c in range(C)] for k in range(K)]
    y = [[[[None] * Wo for _ in range(Ho)] for _ in range(K)] for _ in range(N)]
    for n in range(N):
        for ti in range(th):
            for tj in range(tw):
                Vs = [_mm(_mm(_tr(rb.BP), halo_tile(x[n][c], ti, tj, m, nx, pad)), rb.BP) for c in range(C)]
                for k in range(K):
                    Z = [[Fraction(0)] * rb.D for _ in range(rb.D)]
                    for c in range(C):
                        Zc = residue_bilinear_2d(rb, Us[k][c], Vs[c])
                        Z = [[Z[i][j] + Zc[i][j] for j in range(rb.D)] for i in range(rb.D)]
                    Y = _mm(_mm(_tr(rb.AP), Z), rb.AP)
                    for a in range(m):
                        for b in range(m):
                            i, j = ti * m + a, tj * m + b
                            if i < Ho and j < Wo:
                                y[n][k][i][j] = Y[a][b]
    return y
