"""Small invocations of every kernel family of libwino.so, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

  K2 weight transform (point fast path, residue slabs), K1 input transform (TMA NCHW
  flat and 3D boxes, NHWC TMA, NHWC direct-load, synchronous pairs, tiles > 8x8), K3
  tcgen05 GEMM (kind::f16, 3 x kind::tf32, residue schedule), K4 output transform
  (thread per tile, TMA-staged for domains >= 7, NHWC), the fused split K3+K4 kernel,
  the chunked K3->K4 path, K5 1D tiles, K6 statistics, K7 paper-mode 2D tiles and the
  fp64 direct reference.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import datagen
    import paper_1905_05233_b200 as W
    from paper_1905_05233_b200.algos import canonical_spec
    td = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
    fused = os.environ.get("WINO_FUSED", "")
    cases = [
        # name, lowering, N, C, K, H, W, pad, dtype, layout
        ("lin4", "subsolver", 1, 72, 136, 19, 23, 1, "bf16", "nchw"),    # flat TMA boxes (W*2 % 16 != 0), K3 BN 256
        ("lin4", "subsolver", 1, 64, 64, 16, 32, 1, "fp16", "nchw"),     # 3D TMA boxes, BN 64
        ("sup1_6", "subsolver", 1, 64, 72, 20, 20, 1, "bf16", "nchw"),   # D = 9: TMA-staged K4
        ("lin3", "subsolver", 1, 40, 40, 15, 15, 1, "fp16", "nchw"),     # odd W: synchronous pairs K1
        ("lin4", "subsolver", 1, 64, 64, 16, 16, 1, "fp32", "nchw"),     # 3 x TF32
        ("sup1_4", "residue", 1, 72, 40, 13, 13, 1, "bf16", "nchw"),     # residue slabs + schedule
        ("lin4", "subsolver", 1, 64, 40, 16, 16, 1, "bf16", "nhwc"),     # NHWC TMA K1, NHWC K4
        ("lin2", "subsolver", 1, 3, 16, 18, 18, 1, "bf16", "nhwc"),      # NHWC direct-load K1 (C = 3)
        ("sup1_10", "subsolver", 1, 16, 16, 21, 21, 1, "bf16", "nchw"),  # tiles beyond 8x8
    ]
    for name, low, N, C, K, H, Wd, pad, dt, lay in cases:
        spec, m = canonical_spec(name)
        a = W.WinoAlgo(spec, m, lowering=low)
        x, w = datagen.layer(N, C, K, H, Wd, dt, seed=1)
        xt = torch.from_numpy(x).to(td[dt]).cuda()
        if lay == "nhwc":
            xt = xt.permute(0, 2, 3, 1).contiguous()
        y = W.wino_conv2d(xt, torch.from_numpy(w).to(td[dt]).cuda(), a, pad=pad, layout=lay)
        torch.cuda.synchronize()
        print(name, low, dt, lay, "launches", W.wino_last_launch_count(), "finite", bool(torch.isfinite(y).all()),
              flush=True)
    # fused split K3 + K4 (K > 128, 16-bit, NCHW), run when WINO_FUSED=1
    if fused == "1":
        for name in ("lin4", "sup1_6"):
            spec, m = canonical_spec(name)
            a = W.WinoAlgo(spec, m)
            x, w = datagen.layer(2, 64, 272, 23, 19, "bf16", seed=2)
            y = W.wino_conv2d(torch.from_numpy(x).to(torch.bfloat16).cuda(),
                              torch.from_numpy(w).to(torch.bfloat16).cuda(), a)
            torch.cuda.synchronize()
            print("fused", name, bool(torch.isfinite(y).all()), flush=True)
    # K5 / K6 / K7 / direct f64
    spec, m = canonical_spec("sup1_6")
    a = W.WinoAlgo(spec, m)
    xx, hh = datagen.tiles1d(1000, m, "fp16", seed=3)
    W.wino_conv1d_tiles(torch.from_numpy(xx).half().cuda(), torch.from_numpy(hh).half().cuda(), a, True)
    d = torch.randn(5, 100, m + 2, m + 2, device="cuda").half()
    g = torch.randn(5, 100, 3, 3, device="cuda").half()
    for csum in ("sequential", "pairwise"):
        W.wino_conv2d_tiles_paper(d, g, a, csum, "fp32")
    x, w = datagen.layer(1, 16, 8, 13, 13, "bf16", seed=4)
    xt, wt = torch.from_numpy(x).to(torch.bfloat16).cuda(), torch.from_numpy(w).to(torch.bfloat16).cuda()
    yref = W.wino_direct_conv2d_f64(xt, wt, 1)
    y = W.wino_conv2d(xt, wt, a)
    print("stats", W.summary(W.wino_error_stats(y, yref, m).cpu()), flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
