"""GPU parity: libwino's CUDA path (through the C ABI) against the CPU oracle.

Bars:
* every stage (U, V, M, y) element by element against the oracle's pipeline
  model fed the same inputs, within the dtype rounding of fp32 values computed
  in a different order (at most one dtype ulp apart plus fp32 slack);
* the whole layer element by element against fp64 direct convolution within
  the a-priori forward error bound of the pipeline model;
* fp32: relative L1 <= 1e-4 (m <= 4), <= 1e-3 (m <= 8) (north star);
* fp16 / bf16: mean per-tile relative error within +-10% of the oracle's
  emulated error for the same algorithm and inputs, identical ranking;
* 1D tiles in paper mode: bitwise equal to the oracle;
* error statistics / fp64 direct kernels: 1e-12 relative.
"""
import os
import numpy as np
import pytest
import torch

import datagen
import paper_1905_05233_b200 as W
from oracle import conv as CV
from oracle import metrics as MT
from oracle import precision as P
from oracle import transforms as T

pytestmark = pytest.mark.gpu

TD = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
U_D = {"fp32": 2.0 ** -24, "fp16": 2.0 ** -11, "bf16": 2.0 ** -8}


def dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(TD[dtype]).cuda()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64) if t.dtype != torch.float64 else t.cpu().numpy()


def algo_pair(name, lowering="subsolver"):
    mods, m = T.canonical(name)
    spec = T.moduli_spec(mods)
    a = W.WinoAlgo(spec, m, lowering=lowering)
    ref = T.make_transforms(mods, m) if lowering == "subsolver" else T.residue_blocks(mods, m)
    return a, ref, m


def close_to_rounded(got, want, dtype, scale):
    """got, want: dtype values of the same fp32 quantity computed in different
    orders.  They may differ by one dtype ulp where the fp32 values straddle a
    rounding boundary, plus the fp32 order difference itself (scale = the
    magnitude bound of the summands)."""
    tol = 2.0 * U_D[dtype] * np.abs(want) + 64 * 2.0 ** -24 * scale + 1e-30
    bad = np.abs(got - want) > tol
    assert not bad.any(), (int(bad.sum()), float(np.abs(got - want).max()))
    return float((got == want).mean())


# ------------------------------------------------------------------ stages


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("name,lowering", [("lin4", "subsolver"), ("sup1_4", "subsolver"), ("sup1_6", "residue"),
                                           ("sup2_4", "residue"), ("lin8", "subsolver")])
def test_weight_transform(dtype, name, lowering):
    a, ref, m = algo_pair(name, lowering)
    K, C = 24, 72
    _, w = datagen.layer(1, C, K, 4, 4, dtype, seed=3)
    U = W.wino_weight_transform(dev(w, dtype), a)
    torch.cuda.synchronize()
    if lowering == "subsolver":
        Uo = P.pipeline_weight_transform(ref, w, dtype).reshape(a.units, K, C)
        absG = np.abs(np.array([[float(v) for v in r] for r in ref.G]))
    else:
        _, Uo = P.pipeline_residue_weights(ref, w, dtype)
        absG = np.abs(np.array([[float(v) for v in r] for r in ref.GP])) * 2
    got = host(U[0]) + (host(U[1]) if dtype == "fp32" else 0)
    scale = P.sep2(absG, np.abs(w).transpose(2, 3, 0, 1)).reshape(-1, K, C).max()
    if dtype == "fp32":
        assert np.abs(got[:, :, :C] - Uo).max() <= 2.0 ** -20 * scale
    else:
        close_to_rounded(got[:, :, :C], Uo, dtype, scale)
    assert not got[:, :, C:].any()                      # channel padding is zero


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("name,lowering,pad", [("lin4", "subsolver", 1), ("sup1_6", "subsolver", 1),
                                               ("lin3", "subsolver", 0), ("sup1_4", "residue", 1),
                                               ("lin8", "subsolver", 1)])
@pytest.mark.parametrize("shape", [(2, 40, 19, 23), (2, 40, 28, 28), (1, 72, 18, 32), (2, 8, 14, 14),
                                   (3, 128, 28, 28)],
                         ids=["odd-sync", "w28-flat16-3d32", "w32-3d", "w14-flat", "w28-c128"])
def test_input_transform(dtype, name, lowering, pad, shape):
    """K1 vs the oracle's pipeline-mode V (rd(B^T d B), Eq. 2) on shapes that
    reach each staging path: odd planes (synchronous), W*es % 16 != 0 with whole
    rows (TMA flat boxes; row-group boxes when a step's rows exceed 256 elements,
    lin8 at W = 28 in 16 bits), W*es % 16 == 0 (TMA 3D boxes), channels < 64, and
    full 64-channel blocks over several persistent work items (vector converter)."""
    a, ref, m = algo_pair(name, lowering)
    N, C, H, Wd = shape
    x, _ = datagen.layer(N, C, 1, H, Wd, dtype, seed=4)
    V = W.wino_input_transform(dev(x, dtype), a, pad=pad)
    torch.cuda.synchronize()
    T_all = CV.tile_grid(H, Wd, m, pad)
    V = W.v_to_dense(V, N * T_all[2] * T_all[3])
    D = a.domain
    if lowering == "subsolver":
        Vo, _ = P.pipeline_input_transform(ref, x, dtype, pad)
        absBT = np.abs(np.array([[float(v) for v in r] for r in ref.BT]))
    else:
        BPT = P.lower_f32([list(r) for r in zip(*ref.BP)])
        d, _ = P.halo_tiles(np.asarray(x, np.float32), m, m + 2, pad)
        Vo = P.rd(dtype, P.sep2(BPT, d)).transpose(0, 1, 2, 4, 5, 3).reshape(D, D, -1, C)
        absBT = np.abs(BPT.astype(np.float64))
    Vo = Vo.reshape(D * D, -1, C)
    got = host(V[0]) + (host(V[1]) if dtype == "fp32" else 0)
    assert got.shape[1] == Vo.shape[1]
    scale = (absBT.sum(1).max() ** 2) * np.abs(x).max()
    if dtype == "fp32":
        assert np.abs(got[:, :, :C] - Vo).max() <= 2.0 ** -20 * scale
    else:
        frac = close_to_rounded(got[:, :, :C], Vo, dtype, scale)
        assert frac > 0.99
    assert not got[:, :, C:].any()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name,lowering,T_,C,K", [("lin4", "subsolver", 300, 136, 72),
                                                  ("lin2", "subsolver", 129, 64, 256),
                                                  ("sup1_4", "residue", 257, 70, 40),
                                                  ("lin4", "subsolver", 1000, 512, 512),
                                                  # CTA-pair K3 (K > 128): odd tile-block count, half-empty k tile
                                                  ("lin4", "subsolver", 300, 136, 384),
                                                  ("sup1_4", "residue", 383, 70, 200)])
def test_domain_gemm_isolated(dtype, name, lowering, T_, C, K):
    """Feed identical U, V (oracle-made, dtype values) to the tensor-core GEMM."""
    a, ref, m = algo_pair(name, lowering)
    rng = np.random.default_rng(7)
    Q, S = a.domain ** 2, a.units
    Cp = -(-C // 64) * 64
    Vh = np.zeros((1, Q, T_, Cp))
    Uh = np.zeros((1, S, K, Cp))
    Vh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, Q, T_, C)), dtype)
    Uh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, S, K, C)), dtype)
    M = W.wino_domain_gemm(W.v_from_dense(dev(Vh, dtype)), dev(Uh, dtype), a, C, K, T_)
    torch.cuda.synchronize()
    got = host(M)[:, :, :T_]
    # the unit -> (output point, input point) pairs come from the oracle (O6), and
    # the library's schedule must list the same units in the same order
    if lowering == "subsolver":
        pairs = [(q, q) for q in range(Q)]
    else:
        pairs = [(po, pi) for (po, pi, *_r) in P.residue_slabs(ref)]
    out_pt, in_pt = [p[0] for p in pairs], [p[1] for p in pairs]
    lib_out, lib_in, *_ = a.unit_table()
    assert list(lib_out) == out_pt and list(lib_in) == in_pt
    want = np.zeros((Q, K, T_))
    aw = np.zeros((Q, K, T_))
    for u in range(S):
        want[out_pt[u]] += Uh[0, u] @ Vh[0, in_pt[u]].T
        aw[out_pt[u]] += np.abs(Uh[0, u]) @ np.abs(Vh[0, in_pt[u]]).T
    # fp32 accumulation of exact products: |err| <= gamma_n * sum |u v|
    n = C * max(1, S // Q)
    assert (np.abs(got - want) <= 1.01 * n * 2.0 ** -24 * aw + 1e-30).all()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("T_,K", [(300, 384), (1000, 512), (129, 256)])
def test_domain_gemm_pair_equals_single(dtype, T_, K, monkeypatch):
    """The CTA-pair K3 (cta_group::2, default for K > 128) and the one-CTA kernel
    (WINO_PAIR=0) run the same fp32 accumulation: identical bits."""
    a, ref, m = algo_pair("lin4")
    rng = np.random.default_rng(11)
    Q, C = a.domain ** 2, 200
    Cp = -(-C // 64) * 64
    Vh = np.zeros((1, Q, T_, Cp))
    Uh = np.zeros((1, Q, K, Cp))
    Vh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, Q, T_, C)), dtype)
    Uh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, Q, K, C)), dtype)
    Vd, Ud = W.v_from_dense(dev(Vh, dtype)), dev(Uh, dtype)
    M2 = W.wino_domain_gemm(Vd, Ud, a, C, K, T_)
    monkeypatch.setenv("WINO_PAIR", "0")
    M1 = W.wino_domain_gemm(Vd, Ud, a, C, K, T_)
    torch.cuda.synchronize()
    assert torch.equal(M1[:, :, :T_], M2[:, :, :T_])


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("T_,K,C,m_store", [(1000, 512, 200, "fp32"), (300, 384, 512, "fp32"), (1000, 512, 136, "dtype"),
                                          (129, 260, 64, "fp32")])
def test_domain_gemm_resident_u_equals_streamed(dtype, T_, K, C, m_store, monkeypatch):
    """The resident-U CTA-pair K3 (opt-in WINO_URES=1: U slice kept in shared
    memory, 16-bit SUBSOLVER layers with Cp <= 512) and the default streamed-U
    pair kernel accumulate in the same order: identical bits, fp32 or 16-bit M."""
    a, ref, m = algo_pair("lin4")
    if m_store == "dtype":
        a.set_m_storage("dtype")
    rng = np.random.default_rng(13)
    Q = a.domain ** 2
    Cp = -(-C // 64) * 64
    Vh = np.zeros((1, Q, T_, Cp))
    Uh = np.zeros((1, Q, K, Cp))
    Vh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, Q, T_, C)), dtype)
    Uh[..., :C] = datagen.to_dtype_values(rng.standard_normal((1, Q, K, C)), dtype)
    Vd, Ud = W.v_from_dense(dev(Vh, dtype)), dev(Uh, dtype)
    M2 = W.wino_domain_gemm(Vd, Ud, a, C, K, T_)
    monkeypatch.setenv("WINO_URES", "1")
    M1 = W.wino_domain_gemm(Vd, Ud, a, C, K, T_)
    torch.cuda.synchronize()
    assert torch.equal(M1[:, :, :T_], M2[:, :, :T_])


def test_domain_gemm_pair_equals_single_tf32(monkeypatch):
    """fp32 (3xTF32 from hi/lo planes): the CTA-pair K3 equals the one-CTA kernel bitwise."""
    a, ref, m = algo_pair("lin4")
    x, w = datagen.layer(3, 96, 200, 22, 26, "fp32", seed=6)
    U = W.wino_weight_transform(dev(w, "fp32"), a)
    V = W.wino_input_transform(dev(x, "fp32"), a)
    T_all = CV.tile_grid(22, 26, 4, 1)
    T0 = 3 * T_all[2] * T_all[3]
    M2 = W.wino_domain_gemm(V, U, a, 96, 200, T0)
    monkeypatch.setenv("WINO_PAIR", "0")
    M1 = W.wino_domain_gemm(V, U, a, 96, 200, T0)
    torch.cuda.synchronize()
    assert torch.equal(M1[:, :, :T0], M2[:, :, :T0])


def test_domain_gemm_tf32x3():
    """fp32 path: U, V made by the library (hi/lo planes); M vs fp64 products."""
    a, ref, m = algo_pair("lin4")
    x, w = datagen.layer(1, 96, 48, 14, 18, "fp32", seed=5)
    xd, wd = dev(x, "fp32"), dev(w, "fp32")
    U = W.wino_weight_transform(wd, a)
    V = W.wino_input_transform(xd, a)
    T_all = CV.tile_grid(14, 18, 4, 1)
    T0 = T_all[2] * T_all[3]
    M = W.wino_domain_gemm(V, U, a, 96, 48, T0)
    torch.cuda.synchronize()
    V = W.v_to_dense(V, T0)
    Uf = (host(U[0]) + host(U[1]))[:, :, :96]
    Vf = (host(V[0]) + host(V[1]))[:, :, :96]
    T_ = Vf.shape[1]
    want = np.einsum("qkc,qtc->qkt", Uf, Vf)
    aw = np.einsum("qkc,qtc->qkt", np.abs(Uf), np.abs(Vf))
    got = host(M)[:, :, :T_]
    assert (np.abs(got - want) <= (96 * 2.0 ** -24 + 2.0 ** -20) * aw + 1e-30).all()


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("name,lowering", [("lin4", "subsolver"), ("sup1_6", "subsolver"), ("sup1_4", "residue"),
                                           ("lin5", "subsolver"), ("sup1_7", "subsolver"), ("lin8", "subsolver")])
def test_output_transform(dtype, name, lowering):
    """K4 alone vs the oracle's separable A^T M A on a ragged 17 x 13 output (odd m in
    16-bit: Y staged through shared memory; D = 10: the two-buffer TMA ring)."""
    a, ref, m = algo_pair(name, lowering)
    N, K, H, Wd = 2, 20, 17, 13
    Ho, Wo, th, tw = CV.tile_grid(H, Wd, m, 1)
    T_ = N * th * tw
    rng = np.random.default_rng(8)
    D = a.domain
    Mh = rng.standard_normal((D * D, K, T_)).astype(np.float32)
    Md = torch.zeros((D * D, K, -(-T_ // 32) * 32), dtype=torch.float32)   # Tp: T rounded up to 32
    Md[:, :, :T_] = torch.from_numpy(Mh)
    y = W.wino_output_transform(Md.cuda(), a, N, K, H, Wd, 1, dtype)
    torch.cuda.synchronize()
    AT = P.lower_f32(ref.AT if lowering == "subsolver" else [list(r) for r in zip(*ref.AP)])
    Yt = P.rd(dtype, P.sep2(AT, Mh.reshape(D, D, K, T_)))
    want = P._scatter_tiles(Yt, N, K, th, tw, m, Ho, Wo)
    scale = np.abs(AT).sum(1).max() ** 2 * np.abs(Mh).max()
    close_to_rounded(host(y), want.astype(np.float64), dtype, scale)


# ------------------------------------------------------------------ whole layer


def algo_pair_spec(spec, m, lowering="subsolver"):
    mods = T.parse_moduli(spec)
    a = W.WinoAlgo(spec, m, lowering=lowering)
    ref = T.make_transforms(mods, m) if lowering == "subsolver" else T.residue_blocks(mods, m)
    return a, ref, m


def _layer_check(name, lowering, dtype, N, C, K, H, Wd, pad, xdist="relu_normal", seed=0, m=None):
    a, ref, m = algo_pair(name, lowering) if m is None else algo_pair_spec(name, m, lowering)
    x, w = datagen.layer(N, C, K, H, Wd, dtype, seed=seed, xdist=xdist)
    y = W.wino_conv2d(dev(x, dtype), dev(w, dtype), a, pad=pad)
    assert W.wino_last_launch_count() in (3, 4)   # K2, K1, fused K3+K4 | K3, K4
    torch.cuda.synchronize()
    yg = host(y)
    yref = CV.direct_conv2d_f64(x, w, pad)
    if lowering == "subsolver":
        yo = P.pipeline_conv2d(ref, x, w, dtype, pad)
        bound = P.elementwise_bound(ref, x, w, dtype, yref, pad, mma_rel=2.0 ** -20 if dtype == "fp32" else 0.0)
        bad = np.abs(yg - yref) > bound
        assert not bad.any(), (int(bad.sum()), float(np.abs(yg - yref).max()))
    else:
        yo = P.pipeline_residue_conv2d(ref, x, w, dtype, pad)
        bound = P.residue_elementwise_bound(ref, x, w, dtype, yref, pad,
                                            mma_rel=2.0 ** -20 if dtype == "fp32" else 0.0)
        bad = np.abs(yg - yref) > bound
        assert not bad.any(), (int(bad.sum()), float(np.abs(yg - yref).max()))
    sg = MT.summary(MT.stats8(yg, yref, m))
    so = MT.summary(MT.stats8(yo, yref, m))
    return sg, so, m


LAYER_CASES = [
    ("lin2", "subsolver", 1, 8, 8, 16, 16, 1),          # cfg1 shape
    ("sup1_2", "subsolver", 1, 8, 8, 16, 16, 1),
    ("sup1_3", "subsolver", 1, 8, 8, 16, 16, 1),        # cfg1's literal {a, a+1, a^2+1, inf}
    ("lin4", "subsolver", 2, 72, 40, 19, 23, 1),        # ragged everywhere, C not a multiple of 64
    ("sup1_4", "subsolver", 2, 72, 40, 19, 23, 0),
    ("lin6", "subsolver", 1, 128, 136, 30, 30, 1),
    ("sup1_6", "subsolver", 1, 128, 136, 30, 30, 1),
    ("lin8", "subsolver", 1, 64, 64, 26, 26, 1),
    ("sup1_8", "subsolver", 1, 64, 64, 26, 26, 1),
    ("sup2_6", "subsolver", 1, 64, 64, 26, 26, 1),
    ("sup1_4", "residue", 2, 72, 40, 19, 23, 1),
    ("sup1_6", "residue", 1, 128, 136, 30, 30, 1),
    ("sup2_4", "residue", 1, 64, 48, 20, 20, 1),
    ("lin4", "subsolver", 1, 3, 64, 224, 224, 1),       # VGG conv1_1: C = 3, 224 wide (3D TMA boxes, column blocks)
    ("lin4", "subsolver", 2, 128, 128, 14, 14, 1),      # VGG block 5 spatial size (flat boxes, 4-row alignment)
    ("sup1_6", "subsolver", 1, 64, 72, 56, 56, 1),      # VGG block 3 spatial size, m = 6
    ("sup1_10", "subsolver", 1, 64, 64, 25, 27, 1),     # Table 3 W(10x10), mu = 13
    ("sup1_12", "subsolver", 1, 64, 64, 27, 29, 1),     # Table 3 W(12x12), mu = 15 (reading A21 points)
    ("sup2_12", "subsolver", 1, 64, 64, 26, 26, 1),     # two quadratics at 12x12, mu = 16
]


@pytest.mark.parametrize("case", LAYER_CASES, ids=lambda c: f"{c[0]}-{c[1]}-C{c[3]}K{c[4]}-{c[5]}x{c[6]}p{c[7]}")
@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
def test_layer(case, dtype):
    name, lowering, N, C, K, H, Wd, pad = case
    sg, so, m = _layer_check(name, lowering, dtype, N, C, K, H, Wd, pad)
    if dtype == "fp32":
        assert sg["rel_l1"] <= (1e-4 if m <= 4 else 1e-3), sg
    elif so["nonfinite"] == 0:
        # including the fp16 range-collapse cases (lin8: mean relative error >> 1)
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (sg, so)
    assert sg["nonfinite"] == so["nonfinite"]


HIGHER_DEGREE = [("0,1,a^3+a+1,inf", 4), ("0,a^3-2,inf", 3), ("a^3+a+1,inf", 2), ("0,a^4+1,inf", 4),
                 ("a^4+1,inf", 3), ("a^3+2,a^2+1,inf", 4)]


@pytest.mark.parametrize("spec,m", HIGHER_DEGREE)
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_layer_higher_degree_moduli(spec, m, dtype):
    """Cubic and quartic moduli (Toom-Cook sub-problems on 2d - 1
    points, domain m + 2 + sum(d - 1) up to m + 5): the layer through the C ABI
    against the fp64 direct convolution (element-wise error bound) and the
    oracle's pipeline model."""
    sg, so, _ = _layer_check(spec, "subsolver", dtype, 2, 72, 40, 19, 23, 1, m=m)
    if dtype == "fp32":
        assert sg["rel_l1"] <= 1e-4, sg
    else:
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (sg, so)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_ranking_linear_vs_superlinear(dtype):
    """Ratio-matched pair: F(6x6)+a^2+1 is more accurate than TC F(4x4), on
    the GPU exactly as in the oracle, and within +-10% of it."""
    errs_g, errs_o = {}, {}
    for name in ("lin4", "sup1_6"):
        sg, so, _ = _layer_check(name, "subsolver", dtype, 2, 128, 64, 28, 28, 1, seed=11)
        errs_g[name], errs_o[name] = sg["mean_rel"], so["mean_rel"]
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10
    assert (errs_g["sup1_6"] < errs_g["lin4"]) == (errs_o["sup1_6"] < errs_o["lin4"]) == True  # noqa: E712


def test_ranking_cfg3_full_size():
    """BASELINE cfg3 at full size (N=32, C=K=256, 56x56, fp16): the equal-ratio
    pair of P:596 -- W F(6x6)+a^2+1 more accurate than TC F(4x4) -- on the GPU
    as in the oracle's emulation of the same whole layer, each within +-10 %."""
    c = dict(datagen.CONFIGS["cfg3"])
    x, w = datagen.layer(c["N"], c["C"], c["K"], c["H"], c["W"], "fp16", seed=0, xdist=c["xdist"])
    xd, wd = dev(x, "fp16"), dev(w, "fp16")
    yr = W.wino_direct_conv2d_f64(xd, wd, 1)
    yref = host(yr)
    eg, eo = {}, {}
    for name in ("lin4", "sup1_6"):
        a, ref, m = algo_pair(name)
        eg[name] = W.summary(W.wino_error_stats(W.wino_conv2d(xd, wd, a), yr, m))["mean_rel"]
        eo[name] = MT.summary(MT.stats8(P.pipeline_conv2d(ref, x, w, "fp16"), yref, m))["mean_rel"]
        assert abs(eg[name] / eo[name] - 1) <= 0.10, (name, eg[name], eo[name])
    assert eg["sup1_6"] < eg["lin4"] and eo["sup1_6"] < eo["lin4"]


def test_edge_cases():
    # single output pixel, single channel, pad 0
    for (N, C, K, H, Wd, pad) in [(1, 1, 1, 3, 3, 0), (1, 1, 1, 1, 1, 1), (3, 3, 64, 9, 5, 1), (1, 130, 17, 6, 40, 1)]:
        sg, so, m = _layer_check("lin4", "subsolver", "fp32", N, C, K, H, Wd, pad, xdist="uniform01")
        assert sg["rel_l1"] <= 1e-4


def test_fp16_overflow_is_counted_not_an_error():
    a, ref, m = algo_pair("lin8")
    rng = np.random.default_rng(2)
    x = datagen.to_dtype_values(300.0 * rng.standard_normal((1, 16, 20, 20)), "fp16")
    w = datagen.to_dtype_values(rng.standard_normal((8, 16, 3, 3)), "fp16")
    y = W.wino_conv2d(dev(x, "fp16"), dev(w, "fp16"), a)
    torch.cuda.synchronize()
    yg = host(y)
    yo = P.pipeline_conv2d(ref, x, w, "fp16")
    ng, no = int((~np.isfinite(yg)).sum()), int((~np.isfinite(yo)).sum())
    assert no > 0 and abs(ng - no) <= max(2, 0.02 * no)


# ------------------------------------------------------------------ 1D tiles (cfg 2)


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("fam", ["lin", "sup1", "sup2"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_conv1d_paper_mode_bitwise(dtype, fam, n):
    mods, m = T.canonical(f"{fam}{n}")
    ts = T.make_transforms(mods, m)
    a = W.WinoAlgo(T.moduli_spec(mods), m)
    Tn = (1 << 15) + 3
    x, h = datagen.tiles1d(Tn, n, dtype, seed=n)
    for mode in (("rne", "trunc") if dtype == "bf16" else ("rne",)):
        y = W.wino_conv1d_tiles(dev(x, dtype), dev(h, dtype), a, per_op_rounding=True, bf16_mode=mode)
        torch.cuda.synchronize()
        yo = P.paper_conv1d(ts, x, h, dtype, bf16_mode=mode)
        g = host(y).astype(np.float32)
        same = (g.view(np.uint32) == yo.astype(np.float32).view(np.uint32)) | (np.isnan(g) & np.isnan(yo))
        assert same.all(), (mode, int((~same).sum()))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name", ["lin4", "sup1_6", "sup2_8"])
def test_conv1d_pipeline_mode(dtype, name):
    mods, m = T.canonical(name)
    ts = T.make_transforms(mods, m)
    a = W.WinoAlgo(T.moduli_spec(mods), m)
    x, h = datagen.tiles1d(1 << 14, m, dtype, seed=1)
    y = W.wino_conv1d_tiles(dev(x, dtype), dev(h, dtype), a, per_op_rounding=False)
    torch.cuda.synchronize()
    yo = P.pipeline_conv1d(ts, x, h, dtype)
    ref = np.stack([sum(h[:, k] * x[:, j + k] for k in range(3)) for j in range(m)], 1)
    eg, eo = MT.tile_rel_1d(host(y), ref).mean(), MT.tile_rel_1d(yo, ref).mean()
    assert abs(eg / eo - 1) <= 0.10


# ------------------------------------------------------------------ metric path kernels


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_error_stats_kernel(dtype):
    rng = np.random.default_rng(0)
    N, K, Ho, Wo, m = 2, 5, 13, 11, 4
    yref = rng.standard_normal((N, K, Ho, Wo))
    y = datagen.to_dtype_values(yref + 1e-3 * rng.standard_normal(yref.shape), dtype)
    y[0, 1, 3, 4] = np.inf
    yref[1, 2, :4, :4] = 0
    y[1, 2, :4, :4] = 0
    s = W.wino_error_stats(dev(y, dtype), torch.from_numpy(yref).cuda(), m).cpu().numpy()
    so = MT.stats8(y, yref, m)
    assert s[5] == so[5] == 1 and s[6] == so[6] and s[7] == so[7]
    fin = np.isfinite(so)
    np.testing.assert_allclose(s[fin], so[fin], rtol=1e-12)
    assert np.array_equal(np.isinf(s), np.isinf(so))


def test_error_stats_deterministic():
    rng = np.random.default_rng(1)
    yref = rng.standard_normal((4, 64, 28, 28))
    y = dev(yref + 1e-3, "fp32")
    r = torch.from_numpy(yref).cuda()
    a = W.wino_error_stats(y, r, 4).cpu().numpy()
    b = W.wino_error_stats(y, r, 4).cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
def test_direct_f64_kernel(dtype):
    x, w = datagen.layer(2, 19, 37, 15, 70, dtype, seed=9)
    for pad in (0, 1):
        y = W.wino_direct_conv2d_f64(dev(x, dtype), dev(w, dtype), pad).cpu().numpy()
        np.testing.assert_allclose(y, CV.direct_conv2d_f64(x, w, pad), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ full BASELINE sizes, sampled


@pytest.mark.parametrize("cfg,name,dtype", [("cfg3", "lin4", "fp16"), ("cfg3", "sup1_6", "fp16"),
                                            ("cfg5", "lin4", "bf16"), ("cfg5", "sup1_6", "bf16"),
                                            ("cfg5", "lin4", "fp32")] +
                         [("cfg5", n, d) for n in ("lin5", "lin7", "sup1_3", "sup1_5", "sup1_7")
                          for d in ("fp32", "fp16", "bf16")])
def test_full_size_sampled(cfg, name, dtype):
    """Full BASELINE size in the launch configuration bench.py times; the oracle
    recomputes a sample of images (images are independent)."""
    c = dict(datagen.CONFIGS[cfg])
    a, ref, m = algo_pair(name)
    x, w = datagen.layer(c["N"], c["C"], c["K"], c["H"], c["W"], dtype, seed=0, xdist=c["xdist"])
    xd, wd = dev(x, dtype), dev(w, dtype)
    y = W.wino_conv2d(xd, wd, a)
    yr = W.wino_direct_conv2d_f64(xd, wd, 1)
    sg = W.summary(W.wino_error_stats(y, yr, m))
    torch.cuda.synchronize()
    idx = [0, 1, c["N"] - 1]
    xs = x[idx]
    yo = P.pipeline_conv2d(ref, xs, w, dtype)
    yref = CV.direct_conv2d_f64(xs, w, 1)
    np.testing.assert_allclose(host(yr)[idx], yref, rtol=1e-12, atol=1e-12)
    yg = host(y)[idx]
    bound = P.elementwise_bound(ref, xs, w, dtype, yref, 1, mma_rel=2.0 ** -20 if dtype == "fp32" else 0.0)
    assert (np.abs(yg - yref) <= bound).all()
    so = MT.summary(MT.stats8(yo, yref, m))
    ss = MT.summary(MT.stats8(yg, yref, m))
    if dtype == "fp32":
        assert sg["rel_l1"] <= (1e-4 if m <= 4 else 1e-3)
    else:
        assert abs(ss["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (ss, so)
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.15, (sg, so)   # whole layer vs sample


VGG16_STACK = [(3, 64), (64, 64), "pool", (64, 128), (128, 128), "pool", (128, 256), (256, 256), (256, 256), "pool",
               (256, 512), (512, 512), (512, 512), "pool", (512, 512), (512, 512), (512, 512)]


@pytest.mark.parametrize("name", ["lin4", "sup1_6"])
def test_vgg16_stack_per_layer(name):
    """BASELINE cfg4 in miniature: the 13 conv layers of VGG-16 (channel schedule
    64..512, ReLU after every conv, 2x2 max-pool between blocks; DESIGN.md
    reading A16) on a 1 x 3 x 48 x 48 U[0,1) image with He weights, bf16.  Each
    layer runs on the GPU's own previous activation (chained), and its error is
    compared with the oracle's pipeline emulation on the same input (+-10 %)."""
    dtype = "bf16"
    a, ref, m = algo_pair(name)
    rng = np.random.default_rng(5)
    x = datagen.to_dtype_values(rng.random((1, 3, 48, 48)), dtype)
    act = dev(x, dtype)
    li = 0
    for layer in VGG16_STACK:
        if layer == "pool":
            act = torch.nn.functional.max_pool2d(act, 2)
            continue
        cin, cout = layer
        w = datagen.to_dtype_values(rng.normal(0.0, datagen.he_sigma(cin), (cout, cin, 3, 3)), dtype)
        xin = host(act)
        y = W.wino_conv2d(act, dev(w, dtype), a)
        torch.cuda.synchronize()
        yg = host(y)
        yref = CV.direct_conv2d_f64(xin, w, 1)
        yo = P.pipeline_conv2d(ref, xin, w, dtype)
        sg = MT.summary(MT.stats8(yg, yref, m))
        so = MT.summary(MT.stats8(yo, yref, m))
        assert sg["nonfinite"] == so["nonfinite"] == 0
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (li, cin, cout, sg, so)
        act = torch.relu(y)
        li += 1
    assert li == 13


def test_chunked_layer_matches_one_pass():
    """WINO_CHUNK_TB=<blocks>: K3 -> K4 per slice of tile blocks through one
    L2-resident M slice that K4 discards after reading.  Same fp32 arithmetic per
    output, so y is bit-identical to the one-pass layer (ragged last slice, D < 7
    and D >= 7).  Subprocesses: the switch is read once per process."""
    import os
    import subprocess
    import sys
    import tempfile
    code = r"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import datagen, paper_1905_05233_b200 as W
from paper_1905_05233_b200.algos import canonical_spec
out = []
for name, dt, N in (('lin4', 'bf16', 7), ('sup1_6', 'fp16', 5), ('lin3', 'fp32', 3)):
    spec, m = canonical_spec(name)
    a = W.WinoAlgo(spec, m)
    x, w = datagen.layer(N, 80, 136, 29, 31, dt, seed=4)
    td = {'bf16': torch.bfloat16, 'fp16': torch.float16, 'fp32': torch.float32}[dt]
    y = W.wino_conv2d(torch.from_numpy(x).to(td).cuda(), torch.from_numpy(w).to(td).cuda(), a)
    torch.cuda.synchronize()
    out.append(y.float().cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(out))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for chunk in ("", "2", "1"):
        f = tempfile.NamedTemporaryFile(suffix=".npy", delete=False).name
        env = dict(os.environ)
        env.pop("WINO_CHUNK_TB", None)
        if chunk:
            env["WINO_CHUNK_TB"] = chunk
        r = subprocess.run([sys.executable, "-c", code, f], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1]) and np.array_equal(res[0], res[2])


def test_fused_gemm_output_transform_matches_staged():
    """The fused K3+K4 kernel with split SMs (split.cu: tensor-core CTAs write M
    to L2, CUDA-core CTAs transform and discard it) gives bit-identical y to the
    staged K3 -> K4 pair (same fp32 arithmetic per output; only where M lives
    differs) -- for ragged K (272: a partial 256-channel GEMM block and a partial
    32-channel transform slice), ragged tiles, several tile blocks, and any SM
    split or backpressure distance.  Subprocesses: the switches are read per
    process (WINO_FUSED) or per call (WINO_SPLIT_*)."""
    import subprocess
    import sys
    code = r"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import datagen, paper_1905_05233_b200 as W
from paper_1905_05233_b200.algos import canonical_spec
out = []
for name, dt, N, H, Wd in (('lin4', 'bf16', 3, 23, 19), ('sup1_6', 'fp16', 3, 23, 19), ('lin4', 'bf16', 8, 40, 37),
                           ('sup1_6', 'bf16', 8, 41, 40), ('lin2', 'fp16', 4, 30, 30), ('lin8', 'bf16', 4, 33, 35)):
    spec, m = canonical_spec(name)
    a = W.WinoAlgo(spec, m)
    x, w = datagen.layer(N, 96, 272, H, Wd, dt, seed=2)
    td = {'bf16': torch.bfloat16, 'fp16': torch.float16}[dt]
    y = W.wino_conv2d(torch.from_numpy(x).to(td).cuda(), torch.from_numpy(w).to(td).cuda(), a)
    torch.cuda.synchronize()
    out.append(y.float().cpu().numpy())
np.save(sys.argv[1], np.concatenate([o.ravel() for o in out]))
"""
    import os
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    runs = [{"WINO_FUSED": "0"}, {"WINO_FUSED": "1"}, {"WINO_FUSED": "1", "WINO_SPLIT_LAG": "1", "WINO_SPLIT_R": "100"},
            {"WINO_FUSED": "1", "WINO_SPLIT_R": "4", "WINO_SPLIT_LAG": "0"}]
    for extra in runs:
        f = tempfile.NamedTemporaryFile(suffix=".npy", delete=False).name
        env = {k: v for k, v in os.environ.items() if not k.startswith("WINO_")}
        env.update(extra)
        r = subprocess.run([sys.executable, "-c", code, f], cwd=root, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, (extra, r.stderr[-2000:])
        res.append(np.load(f))
    for i in range(1, len(res)):
        assert np.array_equal(res[0], res[i]), runs[i]


NHWC_CASES = [("lin4", "subsolver", 2, 64, 128, 28, 28, 1),     # TMA boxes, 64-channel blocks
              ("lin4", "subsolver", 2, 72, 40, 19, 23, 1),     # ragged, C = 72 (partial channel block)
              ("sup1_6", "subsolver", 1, 128, 136, 30, 30, 1),
              ("lin2", "subsolver", 1, 3, 64, 32, 32, 1),      # C = 3: direct-load fallback
              ("lin8", "subsolver", 1, 64, 64, 26, 26, 0),
              ("sup1_4", "residue", 2, 72, 40, 19, 23, 1),
              ("lin2", "subsolver", 6, 3, 8, 224, 224, 1),     # C = 3 direct-load kernel, T = 75264 > 65535 tiles
              ("sup1_10", "subsolver", 1, 64, 64, 25, 27, 1),  # tiles beyond 8x8 (direct-load K1)
              ("sup1_12", "subsolver", 1, 64, 64, 27, 29, 1)]


@pytest.mark.parametrize("case", NHWC_CASES, ids=lambda c: f"{c[0]}-{c[1]}-C{c[3]}K{c[4]}-{c[5]}x{c[6]}p{c[7]}")
@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
def test_layer_nhwc(case, dtype):
    """NHWC x and y (wino_layout WINO_NHWC): K1 stages channel-contiguous TMA
    boxes with no transpose and K4 writes channel runs through shared memory.
    Same rounding points as NCHW, so y must equal the NCHW result bit for bit,
    and it is checked against the oracle like every layer."""
    name, lowering, N, C, K, H, Wd, pad = case
    a, ref, m = algo_pair(name, lowering)
    x, w = datagen.layer(N, C, K, H, Wd, dtype, seed=9)
    xd, wd = dev(x, dtype), dev(w, dtype)
    y_nchw = W.wino_conv2d(xd, wd, a, pad=pad)
    y_nhwc = W.wino_conv2d(xd.permute(0, 2, 3, 1).contiguous(), wd, a, pad=pad, layout="nhwc")
    torch.cuda.synchronize()
    assert torch.equal(y_nhwc.permute(0, 3, 1, 2), y_nchw)
    yg = host(y_nhwc.permute(0, 3, 1, 2))
    yref = CV.direct_conv2d_f64(x, w, pad)
    if lowering == "subsolver":
        yo = P.pipeline_conv2d(ref, x, w, dtype, pad)
    else:
        yo = P.pipeline_residue_conv2d(ref, x, w, dtype, pad)
    sg = MT.summary(MT.stats8(yg, yref, m))
    so = MT.summary(MT.stats8(yo, yref, m))
    if dtype == "fp32":
        assert sg["rel_l1"] <= (1e-4 if m <= 4 else 1e-3), sg
    elif so["nonfinite"] == 0:
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (sg, so)


@pytest.mark.parametrize("N,layout", [(19, "nchw"), (3, "nchw"), (9, "nhwc")])
def test_host_io_chunked_equals_device_call(N, layout):
    """wino_conv2d_host_io (pinned host x -> device -> layer -> pinned host y,
    processed in up to 8 image chunks with the copies overlapping the layer)
    returns exactly the device call's y, for ragged chunk splits."""
    a, ref, m = algo_pair("lin4")
    x, w = datagen.layer(N, 64, 136, 14, 18, "bf16", seed=12)
    xd, wd = dev(x, "bf16"), dev(w, "bf16")
    if layout == "nhwc":
        xd = xd.permute(0, 2, 3, 1).contiguous()
    y_dev = W.wino_conv2d(xd, wd, a, layout=layout)
    xh = torch.empty(xd.shape, dtype=xd.dtype, pin_memory=True)
    xh.copy_(xd.cpu())
    x2 = torch.empty_like(xd)
    y2 = torch.empty_like(y_dev)
    yh = torch.empty(y_dev.shape, dtype=y_dev.dtype, pin_memory=True)
    yh.zero_()
    ws = W.alloc_workspace(W.wino_conv2d_workspace(a, N, 64, 14, 18, 136, 1, "bf16", layout))
    W.wino_conv2d_host_io(xh, x2, wd, a, y2, yh, ws, layout=layout)
    torch.cuda.synchronize()
    assert torch.equal(yh, y_dev.cpu())


def _error_study():
    import importlib.util
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("error_study", os.path.join(root, "scripts", "error_study.py"))
    es = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(es)
    return es


def test_error_study_trends_on_gpu():
    """Sec. 3.1 / Figure 1 on the GPU path (scripts/error_study.py,
    5000 random trials, each with its own kernel and tile, as P:531): fp32 error
    of the Toom-Cook sets grows with the tile size in 1D and 2D, and at
    the 2D ratio 2.25 the a^2+1 set W F(6x6) beats TC F(4x4) --
    in the paper's per-op rounding and in the tensor-core layer."""
    es = _error_study()
    rows = es.run(5000, dtypes=("fp32",), ns=(2, 4, 6, 8))
    err = {(r["dim"], r["mode"], r["family"], r["n"]): r["mean_euclid"] for r in rows}
    for dim, mode in ((1, "paper"), (2, "paper"), (2, "pipeline")):
        lin = [err[(dim, mode, "lin", n)] for n in (2, 4, 6, 8)]
        assert all(a < b for a, b in zip(lin, lin[1:])), (dim, mode, lin)
    for mode in ("paper", "pipeline"):
        assert err[(2, mode, "sup1[a^2+1]", 6)] < err[(2, mode, "lin", 4)], mode


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_error_study_matches_oracle(dtype):
    """The GPU study's 2D numbers are the oracle's on the same trials: paper mode
    bit for bit (K7 = oracle paper_conv2d_tiles), the pipeline-mode layer within
    +-10 % of the oracle's pipeline emulation per point set (fresh kernel per
    trial)."""
    es = _error_study()
    n, trials = 4, 640
    d, g = es.trials2d(trials, n, 123)
    dd, gd = datagen.to_dtype_values(d, dtype), datagen.to_dtype_values(g, dtype)
    ref = es.direct2d(dd, gd)
    td = TD[dtype]
    for fam, spec in es.point_sets(n):
        a = W.WinoAlgo(spec, n)
        mods = T.parse_moduli(spec)
        ts = T.make_transforms(mods, n)
        yg = W.wino_conv2d_tiles_paper(torch.from_numpy(dd).to(td).cuda(), torch.from_numpy(gd).to(td).cuda(), a)
        yo = P.paper_conv2d_tiles(ts, dd, gd, dtype)
        assert es.errs(host(yg), ref) == es.errs(yo.astype(np.float64), ref), fam
        yp = es.pipeline_diag(W, a, dd, gd, td)
        yop = np.stack([P.pipeline_conv2d(ts, dd[:, s][None], gd[:, s][None], dtype, pad=0)[0, 0]
                        for s in range(trials)])
        eg, eo = es.errs(yp, ref)[0], es.errs(yop.astype(np.float64), ref)[0]
        assert abs(eg / eo - 1) <= 0.10, (fam, eg, eo)


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("name", ["lin4", "sup1_6", "lin8", "sup2_6", "lin2"])
@pytest.mark.parametrize("C", [1, 5, 37])
def test_conv2d_tiles_paper_bitwise(dtype, name, C):
    """K7 (paper-mode multi-channel 2D tiles) equals the oracle's
    paper_conv2d_tiles bit for bit in every channel-sum variant of P:611:
    sequential / pairwise, dtype / fp32 accumulation."""
    mods, m = T.canonical(name)
    ts = T.make_transforms(mods, m)
    a = W.WinoAlgo(T.moduli_spec(mods), m)
    rng = np.random.default_rng(C)
    S = 257
    d = datagen.to_dtype_values(rng.normal(0, 1, (C, S, m + 2, m + 2)), dtype)
    g = datagen.to_dtype_values(rng.normal(0, 1, (C, S, 3, 3)), dtype)
    dd, gd = dev(d, dtype), dev(g, dtype)
    for csum in ("sequential", "pairwise"):
        for acc in ("dtype", "fp32"):
            for mode in (("rne", "trunc") if dtype == "bf16" else ("rne",)):
                y = host(W.wino_conv2d_tiles_paper(dd, gd, a, csum, acc, bf16_mode=mode)).astype(np.float32)
                yo = P.paper_conv2d_tiles(ts, d, g, dtype, bf16_mode=mode, csum=csum, acc=acc).astype(np.float32)
                same = (y.view(np.uint32) == yo.view(np.uint32)) | (np.isnan(y) & np.isnan(yo))
                assert same.all(), (csum, acc, mode, int((~same).sum()))


@pytest.mark.parametrize("name,dtype", [("lin8", "fp16"), ("lin8", "bf16"), ("lin6", "fp16"), ("sup1_8", "fp16")])
def test_layer_scaled_transforms(name, dtype):
    """Power-of-two point balancing on the GPU path (wino_scale_transforms):
    the layer matches the oracle's pipeline emulation of the *scaled* matrices
    within +-10 %, and for fp16 Toom-Cook F(8x8) it removes the range collapse
    of the unscaled algorithm."""
    mods, m = T.canonical(name)
    a = W.WinoAlgo(T.moduli_spec(mods), m).scale("pow2")
    tss = T.scale_pow2_balance(T.make_transforms(mods, m))
    x, w = datagen.layer(1, 64, 136, 26, 26, dtype, seed=21)
    y = W.wino_conv2d(dev(x, dtype), dev(w, dtype), a)
    torch.cuda.synchronize()
    yref = CV.direct_conv2d_f64(x, w, 1)
    sg = MT.summary(MT.stats8(host(y), yref, m))
    so = MT.summary(MT.stats8(P.pipeline_conv2d(tss, x, w, dtype), yref, m))
    assert sg["nonfinite"] == so["nonfinite"] == 0
    assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (sg, so)
    if name == "lin8" and dtype == "fp16":
        y0 = W.wino_conv2d(dev(x, dtype), dev(w, dtype), algo_pair(name)[0])
        torch.cuda.synchronize()
        s0 = MT.summary(MT.stats8(host(y0), yref, m))
        assert s0["mean_rel"] > 10 * sg["mean_rel"], (s0, sg)


# --------------------------------------------------------------------------- M stored in the dtype (reading M3)


def _m3(name, lowering="subsolver"):
    a, ref, m = algo_pair(name, lowering)
    a.set_m_storage("dtype")
    return a, ref, m


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name,lowering,N,H,K", [("lin4", "subsolver", 16, 30, 512), ("lin4", "subsolver", 5, 30, 72),
                                                 ("sup1_4", "residue", 5, 30, 136)])
def test_domain_gemm_m_dtype_is_rounded_accumulator(dtype, name, lowering, N, H, K):
    """K3 under WINO_M_DTYPE stores rd(M) of the same fp32 accumulation: bit for
    bit the RNE cast of the fp32-M kernel's output (CTA-pair and one-CTA)."""
    a32, _, m = algo_pair(name, lowering)
    a16, _, _ = _m3(name, lowering)
    x, w = datagen.layer(N, 136, K, H, H, dtype, seed=21)
    U = W.wino_weight_transform(dev(w, dtype), a32)
    V = W.wino_input_transform(dev(x, dtype), a32)
    T_ = W.geometry(a32, N, 136, H, H, K, 1, dtype)["T"]
    M32 = W.wino_domain_gemm(V, U, a32, 136, K, T_)
    M16 = W.wino_domain_gemm(V, U, a16, 136, K, T_)
    torch.cuda.synchronize()
    assert M16.dtype == TD[dtype]
    assert torch.equal(M16[:, :, :T_], M32[:, :, :T_].to(TD[dtype]))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("name,layout", [("lin4", "nchw"), ("lin3", "nchw"), ("sup1_4", "nchw")])
def test_output_transform_tma_equals_thread_per_tile(dtype, name, layout, monkeypatch):
    """fp32 M: the TMA-staged K4 (default) and the thread-per-tile kernel
    (WINO_K4_TMA32=0, read once per process, so the switch runs in a subprocess)
    apply the same fp32 operations in the same order: identical bits."""
    import subprocess
    import sys
    a32, _, m = algo_pair(name)
    N, K, H = 2, 72, 22
    g = W.geometry(a32, N, 1, H, H, K, 1, dtype)
    rng = np.random.default_rng(7)
    M = rng.standard_normal((a32.domain ** 2, K, g["Tp"])).astype(np.float32)
    y_tma = W.wino_output_transform(torch.from_numpy(M).cuda(), a32, N, K, H, H, 1, dtype, layout=layout)
    torch.cuda.synchronize()
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import paper_1905_05233_b200 as W\n"
        "from paper_1905_05233_b200.algos import canonical_spec\n"
        "s, m = canonical_spec(%r); a = W.WinoAlgo(s, m)\n"
        "M = torch.from_numpy(np.load(sys.argv[1])).cuda()\n"
        "y = W.wino_output_transform(M, a, %d, %d, %d, %d, 1, %r, layout=%r)\n"
        "np.save(sys.argv[2], y.float().cpu().numpy())\n" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                             name, N, K, H, H, dtype, layout))
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        np.save(os.path.join(td, "M.npy"), M)
        env = dict(os.environ, WINO_K4_TMA32="0")
        subprocess.run([sys.executable, "-c", code, os.path.join(td, "M.npy"), os.path.join(td, "y.npy")],
                       check=True, env=env)
        y_tpt = np.load(os.path.join(td, "y.npy"))
    assert np.array_equal(y_tma.float().cpu().numpy(), y_tpt)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name,layout", [("lin4", "nchw"), ("lin6", "nchw"), ("sup1_6", "nchw"), ("lin4", "nhwc")])
def test_output_transform_m_dtype_equals_widened(dtype, name, layout):
    """K4 reading a 16-bit M (thread-per-tile, TMA-staged for domains >= 7, NHWC)
    computes exactly what the fp32-M K4 computes on the widened values."""
    a32, _, m = algo_pair(name)
    a16, _, _ = _m3(name)
    N, K, H = 2, 72, 22
    g = W.geometry(a32, N, 1, H, H, K, 1, dtype)
    rng = np.random.default_rng(5)
    M16 = torch.from_numpy(rng.standard_normal((a32.domain ** 2, K, g["Tp"]))).to(TD[dtype]).cuda()
    y16 = W.wino_output_transform(M16, a16, N, K, H, H, 1, dtype, layout=layout)
    y32 = W.wino_output_transform(M16.float(), a32, N, K, H, H, 1, dtype, layout=layout)
    torch.cuda.synchronize()
    assert torch.equal(y16, y32)


M3_CASES = [("lin2", "subsolver", 1, 8, 8, 16, 16, 1),
            ("lin4", "subsolver", 2, 72, 40, 19, 23, 1),
            ("sup1_4", "subsolver", 2, 72, 40, 19, 23, 0),
            ("lin6", "subsolver", 1, 128, 136, 30, 30, 1),
            ("sup1_6", "subsolver", 1, 128, 136, 30, 30, 1),
            ("lin8", "subsolver", 1, 64, 64, 26, 26, 1),
            ("sup1_4", "residue", 2, 72, 40, 19, 23, 1),
            ("sup1_6", "residue", 1, 128, 136, 30, 30, 1),
            ("lin4", "subsolver", 2, 128, 320, 28, 28, 1),      # K > 256: CTA-pair K3, ragged last pair tile
            ("sup1_10", "subsolver", 1, 64, 64, 25, 27, 1)]


@pytest.mark.parametrize("case", M3_CASES, ids=lambda c: f"{c[0]}-{c[1]}-C{c[3]}K{c[4]}-{c[5]}x{c[6]}p{c[7]}")
@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_layer_m_dtype(case, dtype):
    """Whole layers with M in the dtype (reading M3) against the oracle's
    m_store="dtype" pipeline: inside its elementwise forward bound, mean
    relative error within +-10 %, the same non-finite count."""
    name, lowering, N, C, K, H, Wd, pad = case
    a, ref, m = _m3(name, lowering)
    ms = "dtype" if m <= 8 else "fp32"   # tiles beyond 8x8 keep an fp32 M (include/wino.h)
    x, w = datagen.layer(N, C, K, H, Wd, dtype, seed=4)
    y = W.wino_conv2d(dev(x, dtype), dev(w, dtype), a, pad=pad)
    torch.cuda.synchronize()
    yg = host(y)
    yref = CV.direct_conv2d_f64(x, w, pad)
    if lowering == "subsolver":
        yo = P.pipeline_conv2d(ref, x, w, dtype, pad, m_store=ms)
        bound = P.elementwise_bound(ref, x, w, dtype, yref, pad, m_store=ms)
    else:
        yo = P.pipeline_residue_conv2d(ref, x, w, dtype, pad, m_store=ms)
        bound = P.residue_elementwise_bound(ref, x, w, dtype, yref, pad, m_store=ms)
    fin = np.isfinite(yo)
    bad = (np.abs(yg - yref) > bound) & fin
    assert not bad.any(), (int(bad.sum()), float(np.abs(yg - yref)[fin].max()))
    sg = MT.summary(MT.stats8(yg, yref, m))
    so = MT.summary(MT.stats8(yo, yref, m))
    assert sg["nonfinite"] == so["nonfinite"]
    if so["nonfinite"] == 0:
        assert abs(sg["mean_rel"] / so["mean_rel"] - 1) <= 0.10, (sg, so)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_layer_m_dtype_nhwc_equals_nchw(dtype):
    a, _, m = _m3("lin4")
    x, w = datagen.layer(2, 64, 128, 28, 28, dtype, seed=8)
    xd, wd = dev(x, dtype), dev(w, dtype)
    y1 = W.wino_conv2d(xd, wd, a)
    y2 = W.wino_conv2d(xd.permute(0, 2, 3, 1).contiguous(), wd, a, layout="nhwc")
    torch.cuda.synchronize()
    assert torch.equal(y2.permute(0, 3, 1, 2), y1)


def test_m_dtype_is_a_no_op_for_fp32():
    a32, _, _ = algo_pair("lin4")
    a16, _, _ = _m3("lin4")
    x, w = datagen.layer(1, 64, 64, 20, 20, "fp32", seed=2)
    y1 = W.wino_conv2d(dev(x, "fp32"), dev(w, "fp32"), a32)
    y2 = W.wino_conv2d(dev(x, "fp32"), dev(w, "fp32"), a16)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


def test_m_dtype_ranking_and_error_growth_fp16():
    """Under M3 the superlinear F(6x6) set keeps beating the equal-ratio Toom-Cook
    F(4x4) in fp16, on the GPU as in the oracle."""
    errs = {}
    for name in ("lin4", "sup1_6"):
        a, ref, m = _m3(name)
        x, w = datagen.layer(2, 128, 64, 28, 28, "fp16", seed=12)
        yg = host(W.wino_conv2d(dev(x, "fp16"), dev(w, "fp16"), a))
        yref = CV.direct_conv2d_f64(x, w, 1)
        yo = P.pipeline_conv2d(ref, x, w, "fp16", 1, m_store="dtype")
        errs[name] = (MT.summary(MT.stats8(yg, yref, m))["mean_rel"], MT.summary(MT.stats8(yo, yref, m))["mean_rel"])
    assert errs["sup1_6"][0] < errs["lin4"][0] and errs["sup1_6"][1] < errs["lin4"][1], errs
