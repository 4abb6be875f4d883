"""Timing of the BASELINE configs other than the headline cfg5, on one GPU:

* cfg1 (N=1, C=K=8, 16x16, fp32): latency of one layer, eager and as a CUDA graph, for the
  three cfg1 algorithms (TC F(2x2), {0, a^2+1, inf}, the literal {a, a+1, a^2+1, inf} F(3x3)).
* cfg2 (2^20 independent 1D tiles, n in {2,4,6,8}, paper per-op rounding, K5): GB/s of the
  compulsory traffic x + h + y against the measured HBM copy peak.  Four input sets rotate so the
  working set (>= 4 x 88 MB at n = 8 fp32) exceeds the 126 MB L2.
* cfg3 (N=32, C=K=256, 56x56, fp16): the equal-ratio pair TC F(4x4) vs W F(6x6)+a^2+1 (ratio 2.25,
  P:513) and W F(4x4)+a^2+1, step time, direct-equivalent TFLOP/s and layer roofline fractions.

    python scripts/configs_timing.py > profiles/configs_r02.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def events_ms(fn, reps, st):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    import numpy as np
    import torch
    import bench
    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    peaks, peak_src = bench.load_peaks()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    td = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}
    out = {"peaks": peak_src}

    # ------------------------------------------------------------------ cfg1: latency
    rows = []
    for spec, m in (("0,1,-1,inf", 2), ("0,a^2+1,inf", 2), ("0,-1,a^2+1,inf", 3)):
        algo = Wn.WinoAlgo(spec, m)
        x64, w64 = datagen.layer(1, 8, 8, 16, 16, "fp32", seed=0, xdist="uniform01")
        x = torch.from_numpy(x64).float().cuda()
        w = torch.from_numpy(w64).float().cuda()
        y = torch.empty((1, 8, 16, 16), device="cuda")
        ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, 1, 8, 16, 16, 8, 1, "fp32"))
        step = lambda: Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)   # noqa: E731
        for _ in range(10):
            step()
        eager = events_ms(step, 200, st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step()
        graph = events_ms(g.replay, 200, st)
        rows.append({"algo": f"{{{spec}}} m={m}", "us_eager": eager * 1e3, "us_graph": graph * 1e3,
                     "launches": Wn.wino_last_launch_count()})
    out["cfg1"] = {"workload": "N=1, C=K=8, 16x16, pad 1, fp32, U[0,1) x, He w", "rows": rows}

    # ------------------------------------------------------------------ cfg2: K5 throughput
    rows = []
    T = 1 << 20
    for n in (2, 4, 6, 8):
        for dt in ("fp32", "fp16", "bf16"):
            sets = []
            for k in range(4):
                x, h = datagen.tiles1d(T, n, dt, seed=100 * n + k)
                sets.append((torch.from_numpy(x).to(td[dt]).cuda(), torch.from_numpy(h).to(td[dt]).cuda()))
            for fam in ("lin", "sup1", "sup2"):
                if fam == "sup2" and n < 3:
                    continue
                spec, m = canonical_spec(f"{fam}{n}")
                algo = Wn.WinoAlgo(spec, m)
                it = [0]

                def call():
                    xs, hs = sets[it[0] % 4]
                    it[0] += 1
                    Wn.wino_conv1d_tiles(xs, hs, algo, per_op_rounding=True, stream=st)
                for _ in range(8):
                    call()
                ms = events_ms(call, 64, st)
                es = 4 if dt == "fp32" else 2
                byts = T * (n + 2 + 3 + n) * es
                rows.append({"algo": f"{fam}{n}", "dtype": dt, "us": ms * 1e3, "bytes": byts,
                             "GB/s": byts / (ms * 1e-3) / 1e9, "frac_hbm": byts / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]})
            del sets
    out["cfg2"] = {"workload": "T = 2^20 1D tiles, x ~ U[0,1), h ~ N(0, 0.3), paper per-op rounding (K5)",
                   "bytes": "x + h + y per launch; 4 input sets rotate (working set > L2)", "rows": rows}

    # ------------------------------------------------------------------ cfg3: fp16 equal-ratio pair
    rows = []
    N, C, K, H, W = 32, 256, 256, 56, 56
    x64, w64 = datagen.layer(N, C, K, H, W, "fp16", seed=0, xdist="relu_normal")
    x = torch.from_numpy(x64).half().cuda()
    w = torch.from_numpy(w64).half().cuda()
    yref = Wn.wino_direct_conv2d_f64(x, w, 1, stream=st)
    for name in ("lin4", "sup1_6", "sup1_4"):
        spec, m = canonical_spec(name)
        algo = Wn.WinoAlgo(spec, m)
        y = torch.empty((N, K, H, W), dtype=torch.float16, device="cuda")
        ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, N, C, H, W, K, 1, "fp16"))
        step = lambda: Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)   # noqa: E731
        for _ in range(5):
            step()
        ms = events_ms(step, 50, st)
        s = Wn.summary(Wn.wino_error_stats(y, yref, m, stream=st).cpu())
        g = Wn.geometry(algo, N, C, H, W, K, 1, "fp16")
        B = bench.layer_bytes(N, C, K, H, W, 2, g)
        fr = bench.layer_fracs(ms, B, 2.0 * g["T"] * C * K * g["S"], "fp16", peaks)
        rows.append({"algo": name, "spec": spec, "mu": algo.mu, "ratio": round(algo.ratio_2d, 4), "ms": ms,
                     "tflops_direct_eq": bench.direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12,
                     "frac_compulsory": fr["frac_compulsory"], "frac_staged": fr["frac_staged"],
                     "mean_rel": s["mean_rel"], "rel_l1": s["rel_l1"]})
    out["cfg3"] = {"workload": "N=32, C=K=256, 56x56, pad 1, fp16, post-ReLU x, He w", "rows": rows}

    # ------------------------------------------------------------------ residue lowering vs sub-solver (cfg5)
    rows = []
    N, C, K, H, W = 256, 512, 512, 28, 28
    x64, w64 = datagen.layer(N, C, K, H, W, "bf16", seed=0, xdist="relu_normal")
    x = torch.from_numpy(x64).to(torch.bfloat16).cuda()
    w = torch.from_numpy(w64).to(torch.bfloat16).cuda()
    del x64
    yref = Wn.wino_direct_conv2d_f64(x, w, 1, stream=st)
    for name in ("sup1_4", "sup1_6", "sup1_8", "sup2_6"):
        spec, m = canonical_spec(name)
        for low in ("subsolver", "residue"):
            algo = Wn.WinoAlgo(spec, m, lowering=low)
            y = torch.empty((N, K, H, W), dtype=torch.bfloat16, device="cuda")
            ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, N, C, H, W, K, 1, "bf16"))
            step = lambda: Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)   # noqa: E731
            for _ in range(3):
                step()
            ms = events_ms(step, 20, st)
            s = Wn.summary(Wn.wino_error_stats(y, yref, m, stream=st).cpu())
            rows.append({"algo": name, "lowering": low, "domain": algo.domain, "gemm_units": algo.units, "ms": ms,
                         "tflops_direct_eq": bench.direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12,
                         "mean_rel": s["mean_rel"]})
            del ws, y
    out["residue_vs_subsolver"] = {"workload": "cfg5 (N=256, C=K=512, 28x28) bf16", "rows": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
