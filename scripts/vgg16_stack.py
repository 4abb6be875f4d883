"""BASELINE cfg4: the VGG-16 conv stack (13 conv 3x3 layers, 64 -> 512 channels,
2x2 max-pool between blocks, ReLU after each conv; reading A16) on a
synthetic batch N=64 of 224x224x3 U[0,1) images with He-normal weights, bf16,
for F(4x4) / F(6x6) linear vs superlinear sets.  Per layer: the Winograd layer
time (CUDA events, wino_conv2d incl. its weight transform) and the error vs the
fp64 direct convolution on the device (on a 2-image sample, chained on the
Winograd activations).  ReLU / max-pool between layers are torch glue, not timed.

Network-level proxy for PAPER.md Tables 2-3 (real top-1 needs
ImageNet and trained weights, out of scope): on the first --proxy images, the
whole Winograd-chained stack + final max-pool feeds a random He-normal
classifier (25088 -> 1000, fp64), and its argmax is compared with the same
network run with fp64 direct convolutions (and, as a baseline for what any
bf16 pipeline loses, with bf16 cuDNN direct convolutions).

    python scripts/vgg16_stack.py [--n 64] [--algos lin4,sup1_4,lin6,sup1_6] > profiles/vgg16_stack_r02.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STACK = [(3, 64), (64, 64), "pool", (64, 128), (128, 128), "pool", (128, 256), (256, 256), (256, 256), "pool",
         (256, 512), (512, 512), (512, 512), "pool", (512, 512), (512, 512), (512, 512)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--algos", default="lin4,sup1_4,lin6,sup1_6")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sample", type=int, default=2)
    ap.add_argument("--proxy", type=int, default=32, help="images for the classifier-argmax proxy (0: off)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"])
    ap.add_argument("--m-store", default="fp32", choices=["fp32", "dtype"],
                    help="M between K3 and K4: fp32 (reading R1) or the 16-bit dtype (reading M3)")
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    peaks, peak_src = bench.load_peaks()
    dt = a.dtype
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16}[dt]
    rng = np.random.default_rng(0)
    x0 = torch.from_numpy(rng.random((a.n, 3, 224, 224))).to(tdt).cuda()
    weights = []
    for layer in STACK:
        if layer != "pool":
            cin, cout = layer
            w = rng.normal(0.0, datagen.he_sigma(cin), (cout, cin, 3, 3))
            weights.append(torch.from_numpy(w).to(tdt).cuda())
    out = {"workload": f"BASELINE cfg4: VGG-16 conv stack, N={a.n}, 224x224x3 U[0,1), He weights, {dt}, "
                       f"error on {a.sample} images vs fp64 direct", "peaks": peak_src, "m_store": a.m_store,
           "roofline_note": "per layer: frac_compulsory = max(GEMM flops / tensor peak, (x + w + y) bytes / HBM) / "
                            "time; frac_staged adds U, V and the fp32 M written and read (this design); the GEMM "
                            "flops count the channels padded to the 64-channel block (C = 3 -> 64); M is fp32 or, with "
                            "--m-store dtype, 16-bit", "algos": {}}
    st = torch.cuda.current_stream()
    finals = {}
    for name in a.algos.split(","):
        spec, m = canonical_spec(name)
        algo = Wn.WinoAlgo(spec, m)
        if a.m_store == "dtype":
            algo.set_m_storage("dtype")
        act = x0
        rows, li, total = [], 0, 0.0
        for layer in STACK:
            if layer == "pool":
                act = torch.nn.functional.max_pool2d(act, 2)
                continue
            w = weights[li]
            N, C, H, W = act.shape
            K = w.shape[0]
            ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, N, C, H, W, K, 1, dt))
            y = torch.empty((N, K, H, W), dtype=tdt, device="cuda")
            Wn.wino_conv2d(act, w, algo, out=y, workspace=ws, stream=st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.reps):
                Wn.wino_conv2d(act, w, algo, out=y, workspace=ws, stream=st)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            total += ms
            xs = act[:a.sample].contiguous()
            yref = Wn.wino_direct_conv2d_f64(xs, w, 1, stream=st)
            s = Wn.summary(Wn.wino_error_stats(y[:a.sample].contiguous(), yref, m, stream=st).cpu())
            flops = 2.0 * N * K * C * 9 * H * W
            g = Wn.geometry(algo, N, C, H, W, K, 1, dt)
            B = bench.layer_bytes(N, C, K, H, W, 2, g)
            fr = bench.layer_fracs(ms, B, 2.0 * g["T"] * g["Cp"] * K * g["S"], dt, peaks)
            rows.append({"layer": li + 1, "C": C, "K": K, "HW": H, "ms": ms, "tflops_direct_eq": flops / ms / 1e9,
                         "frac_compulsory": fr["frac_compulsory"], "frac_staged": fr["frac_staged"],
                         "t_roof_us": fr["t_roof_us"], "t_staged_us": fr["t_staged_us"],
                         "rel_l1": s["rel_l1"], "mean_rel": s["mean_rel"], "nonfinite": s["nonfinite"]})
            del ws, yref
            act = torch.relu(y)
            li += 1
        out["algos"][name] = {"spec": spec, "m": m, "mu": algo.mu, "layers": rows, "total_ms": total}
        if a.proxy:
            finals[name] = torch.nn.functional.max_pool2d(act[:a.proxy], 2).double().flatten(1)
        torch.cuda.empty_cache()
    if a.proxy:
        out["classifier_proxy"] = proxy(a, x0, weights, finals, rng)
    print(json.dumps(out, indent=1))


def direct_chain(x, weights, dtype):
    """The same stack with torch direct convolutions in `dtype` (glue identical)."""
    import torch
    act, li = x.to(dtype), 0
    for layer in STACK:
        if layer == "pool":
            act = torch.nn.functional.max_pool2d(act, 2)
            continue
        act = torch.relu(torch.nn.functional.conv2d(act, weights[li].to(dtype), padding=1))
        li += 1
    return torch.nn.functional.max_pool2d(act, 2).double().flatten(1)


def proxy(a, x0, weights, finals, rng):
    import torch
    import numpy as np
    n = a.proxy
    feat = 512 * 7 * 7
    wfc = torch.from_numpy(rng.normal(0.0, np.sqrt(2.0 / feat), (1000, feat))).cuda()   # He-normal, fan-in feat
    ref = direct_chain(x0[:n], weights, torch.float64) @ wfc.T
    top1_ref = ref.argmax(1)
    res = {"images": n, "classifier": "random He-normal FC 25088 -> 1000 (fp64) after the final max-pool",
           "reference": "fp64 direct convolutions, same bf16 inputs and weights", "rows": {}}
    cands = dict(finals)
    cands[f"direct_{a.dtype}_cudnn"] = direct_chain(x0[:n], weights, x0.dtype)
    for name, f in cands.items():
        lg = f @ wfc.T
        top5 = lg.topk(5, dim=1).indices
        res["rows"][name] = {
            "top1_agree": float((lg.argmax(1) == top1_ref).double().mean()),
            "ref_top1_in_top5": float((top5 == top1_ref[:, None]).any(1).double().mean()),
            "logit_rel_l2": float((lg - ref).norm() / ref.norm()),
        }
    return res


if __name__ == "__main__":
    main()
