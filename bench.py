#!/usr/bin/env python
"""Benchmark of the hot path: one step = one 2D Winograd conv layer through
libwino's C ABI (K2 weight transform, K1 input transform, K3 tcgen05
Winograd-domain GEMM, K4 output transform) over one batch of synthetic input.

Default workload (BASELINE.json configs[4], the largest single-GPU config the
metric is quoted on): N=256, C=K=512, 28x28, pad 1, post-ReLU inputs, He
weights; F(4x4, 3x3) Toom-Cook {0,-1,1,-1/2,1/2,inf} in bf16.  Under torchrun
every rank runs its own N=256 images (weak scaling: the layer partitions over
the batch with no exchange step); the only collective is the
NCCL all-reduce of the error statistics, outside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--algo lin4] [--dtype bf16]
    python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Winograd conv TFLOP/s (direct-equiv) & roofline frac per dtype; rel. error vs fp64"
WORKLOADS = {
    "cfg5": dict(N=256, C=512, K=512, H=28, W=28, xdist="relu_normal",
                 desc="BASELINE cfg5: N=256, C=K=512, H=W=28, 3x3, pad 1, post-ReLU Normal x, He-normal w"),
    "cfg3": dict(N=32, C=256, K=256, H=56, W=56, xdist="relu_normal",
                 desc="BASELINE cfg3: N=32, C=K=256, H=W=56, 3x3, pad 1, post-ReLU Normal x, He-normal w"),
    "cfg1": dict(N=1, C=8, K=8, H=16, W=16, xdist="uniform01",
                 desc="BASELINE cfg1: N=1, C=K=8, H=W=16, 3x3, pad 1, U[0,1) x, He-normal w"),
}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=list(WORKLOADS))
    ap.add_argument("--algo", default="lin4")
    ap.add_argument("--dtype", default="bf16", choices=["fp32", "fp16", "bf16"])
    ap.add_argument("--lowering", default="subsolver", choices=["subsolver", "residue"])
    ap.add_argument("--layout", default="nchw", choices=["nchw", "nhwc"],
                    help="activation layout of x and y (BASELINE's x[N,C,H,W] is nchw)")
    ap.add_argument("--sweep", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--no-extras", action="store_true", help="timed loop only (for ncu launch lists)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {k: float(d[k]) for k in FALLBACK_PEAKS if k in d}, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def direct_flops(N, C, K, Ho, Wo):
    return 2.0 * N * K * C * 9 * Ho * Wo


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        import statistics
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- reference arm (CPU oracle)


def run_reference(a, rank, world):
    if rank != 0:
        return
    import numpy as np
    import datagen
    from oracle import precision as P
    from oracle import transforms as T
    c = WORKLOADS[a.workload]
    mods, m = T.canonical(a.algo)
    ts = T.make_transforms(mods, m)
    x, w = datagen.layer(c["N"], c["C"], c["K"], c["H"], c["W"], a.dtype, seed=0, xdist=c["xdist"])
    Ho, Wo = c["H"], c["W"]
    # calibrate: seconds per image, then size each step so the run stays within ~3 minutes
    t0 = time.perf_counter()
    P.pipeline_conv2d(ts, x[:1], w, a.dtype)
    per_img = time.perf_counter() - t0
    n_img = int(max(1, min(c["N"], 150.0 / max(1, a.steps + a.warmup) / max(per_img, 1e-3))))
    xs = x[:n_img]
    for _ in range(a.warmup):
        P.pipeline_conv2d(ts, xs, w, a.dtype)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        P.pipeline_conv2d(ts, xs, w, a.dtype)
    dt = (time.perf_counter() - t0) / a.steps
    val = direct_flops(n_img, c["C"], c["K"], Ho, Wo) / dt / 1e12
    cores = _cpu_threads()
    sample = f"{n_img} of {c['N']} images of {a.workload} per step (pipeline-mode emulation, numpy/BLAS fp32)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
        "config": {"workload": c["desc"], "algo": f"{a.algo} {{{T.moduli_spec(mods)}}}", "sample": sample},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count()


def cpu_baseline(algo_name, dtype, c, budget_s=20.0):
    """The oracle, as it stands, on a bounded sample of the same workload."""
    import datagen
    from oracle import precision as P
    from oracle import transforms as T
    mods, m = T.canonical(algo_name)
    ts = T.make_transforms(mods, m)
    x, w = datagen.layer(c["N"], c["C"], c["K"], c["H"], c["W"], dtype, seed=0, xdist=c["xdist"])
    t0 = time.perf_counter()
    P.pipeline_conv2d(ts, x[:1], w, dtype)
    per = time.perf_counter() - t0
    n = int(max(1, min(c["N"], budget_s / max(per, 1e-3))))
    t0 = time.perf_counter()
    P.pipeline_conv2d(ts, x[:n], w, dtype)
    dt = time.perf_counter() - t0
    return {"value": direct_flops(n, c["C"], c["K"], c["H"], c["W"]) / dt / 1e12, "unit": "TFLOP/s",
            "cores": _cpu_threads(), "kind": "oracle",
            "sample": f"{n} of {c['N']} images, {dt:.1f} s (pipeline-mode emulation of {algo_name} {dtype})"}


# --------------------------------------------------------------------------- our arm


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = WORKLOADS[a.workload]
    spec, m = canonical_spec(a.algo)
    algo = Wn.WinoAlgo(spec, m, lowering=a.lowering)
    tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[a.dtype]
    from paper_1905_05233_b200 import distributed as D
    nl = c["N"]                     # images per rank (weak scaling)
    N = nl * world                  # global batch
    # rank r draws its own images (seed r); the weights are the seed-0 weights on every rank
    x64, _ = datagen.layer(nl, c["C"], c["K"], c["H"], c["W"], a.dtype, seed=rank, xdist=c["xdist"])
    _, w64 = datagen.layer(nl, c["C"], c["K"], c["H"], c["W"], a.dtype, seed=0, xdist=c["xdist"])
    x = torch.from_numpy(np.ascontiguousarray(x64)).to(tdt).cuda()
    if a.layout == "nhwc":
        x = x.permute(0, 2, 3, 1).contiguous()
    w = torch.from_numpy(w64).to(tdt).cuda()
    del x64
    C, K, H, W = c["C"], c["K"], c["H"], c["W"]
    Ho, Wo = H, W
    y = torch.empty((nl, K, Ho, Wo) if a.layout == "nchw" else (nl, Ho, Wo, K), dtype=tdt, device="cuda")
    ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, nl, C, H, W, K, 1, a.dtype, a.layout))
    st = torch.cuda.current_stream()

    def step():
        Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st, layout=a.layout)
        return Wn.wino_last_launch_count()

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(st)
        for _ in range(a.steps):
            launches += step()
        ev1.record(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / a.steps
    if world > 1:
        ms = D.max_over_ranks(ms, dist, "cuda")
    flops = direct_flops(N, C, K, Ho, Wo)
    value = flops / (ms * 1e-3) / 1e12

    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
           "warmup": max(3, a.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
           "config": {"workload": c["desc"], "algo": f"{a.algo} {{{spec}}} m={m} mu={algo.mu} ratio={algo.ratio_2d:.4g}",
                      "lowering": a.lowering, "layout": a.layout, "global_batch": N, "per_gpu_batch": nl,
                      "parallelism": f"dp{world} (batch-partitioned, no data-path collective)",
                      "l2": "inputs larger than L2 (x %.0f MB, V and M staged through HBM)" % (
                          x.numel() * x.element_size() / 1e6 * world)},
           "gpu_launches": launches, "clocks": clk.summary()}
    if not a.no_extras:
        extras(a, out, algo, x, w, y, ws, st, nl, C, K, H, W, m, world, rank, dist, c, spec)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def extras(a, out, algo, x, w, y, ws, st, nl, C, K, H, W, m, world, rank, dist, c, spec):
    import torch
    import paper_1905_05233_b200 as Wn
    peaks, peak_src = load_peaks()
    # ---------------------------------------------------------------- accuracy vs fp64 direct (device)
    xc = x if a.layout == "nchw" else x.permute(0, 3, 1, 2).contiguous()
    yc = y if a.layout == "nchw" else y.permute(0, 3, 1, 2).contiguous()
    yref = Wn.wino_direct_conv2d_f64(xc, w, 1, stream=st)
    stats = Wn.wino_error_stats(yc, yref, m, stream=st)
    del xc, yc
    if world > 1:
        from paper_1905_05233_b200 import distributed as D
        stats = D.reduce_stats(stats, dist)
    out["accuracy"] = {k: (float(v) if not isinstance(v, int) else v) for k, v in Wn.summary(stats.cpu()).items()}
    del yref
    # ---------------------------------------------------------------- per-kernel breakdown (same stream, events)
    g = Wn.geometry(algo, nl, C, H, W, K, 1, a.dtype)
    es = 4 if a.dtype == "fp32" else 2
    pl = g["planes"]
    U = ws[:0]
    base = ws.data_ptr()
    kern = per_kernel_times(algo, x, w, y, ws, st, nl, C, K, H, W, a.dtype, max(20, a.steps // 4),
                            lay=0 if a.layout == "nchw" else 1)
    T_, Q, S, Cp, Tp = g["T"], g["Q"], g["S"], g["Cp"], g["Tp"]
    xb = x.numel() * x.element_size()
    yb = y.numel() * y.element_size()
    wb = w.numel() * w.element_size()
    Ub = pl * S * K * Cp * es
    Vb = pl * Q * T_ * Cp * es
    Mb = Q * K * T_ * 4
    gemm_flops = 2.0 * T_ * C * K * S * (3 if a.dtype == "fp32" else 1)
    hbm = peaks["hbm_gbs"] * 1e9
    tc_peak = peaks["bf16_tflops"] * 1e12 * (0.5 if a.dtype == "fp32" else 1.0)   # tf32 = bf16 / 2 (nominal ratio)
    info = {
        "weight_transform": {"bytes": wb + Ub, "flops": None},
        "input_transform": {"bytes": xb + Vb, "flops": None},
        "domain_gemm": {"bytes": Vb + Ub + Mb, "flops": gemm_flops},
        "output_transform": {"bytes": Mb + yb, "flops": None},
    }
    kernels = {}
    for k_, ms_ in kern.items():
        d = info[k_]
        t_mem = d["bytes"] / hbm
        t_tc = d["flops"] / tc_peak if d["flops"] else 0.0
        kernels[k_] = {"us": ms_ * 1e3, "algorithmic_bytes": d["bytes"], "GB/s": d["bytes"] / (ms_ * 1e-3) / 1e9,
                       "TFLOP/s": (d["flops"] / (ms_ * 1e-3) / 1e12) if d["flops"] else None,
                       "bound": "tensor" if t_tc > t_mem else "hbm", "frac": max(t_mem, t_tc) / (ms_ * 1e-3)}
    out["kernels"] = kernels
    dom = max(kernels, key=lambda k_: kernels[k_]["us"])
    kd = kernels[dom]
    if kd["bound"] == "tensor":
        ach = info[dom]["flops"] / (kd["us"] * 1e-6) / 1e12
        out["roofline"] = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": tc_peak / 1e12,
                           "unit": "TFLOP/s", "frac": ach / (tc_peak / 1e12), "traffic": ncu_traffic(dom, a),
                           "peak_source": peak_src}
    else:
        ach = info[dom]["bytes"] / (kd["us"] * 1e-6) / 1e9
        out["roofline"] = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                           "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": ncu_traffic(dom, a),
                           "peak_source": peak_src}
    # ---------------------------------------------------------------- layer-level rooflines (north star)
    ms = out["ms_per_step"]
    # per GPU (every rank runs the same per-GPU layer concurrently)
    comp_bytes = xb + yb + wb
    t_roof = max(gemm_flops / tc_peak, comp_bytes / hbm)
    t_staged = max(gemm_flops / tc_peak, (comp_bytes + Ub + 2 * Vb + 2 * Mb) / hbm)
    out["layer_roofline"] = {"t_roof_us": t_roof * 1e6, "frac_compulsory": t_roof / (ms * 1e-3),
                             "t_staged_us": t_staged * 1e6, "frac_staged": t_staged / (ms * 1e-3),
                             "peaks": peak_src}
    # ---------------------------------------------------------------- end to end (host buffers)
    out["e2e"] = e2e(algo, x, w, y, ws, st, nl, C, K, H, W, a, world, dist)
    # ---------------------------------------------------------------- CPU baseline (rank 0, N=1 only)
    if world == 1:
        out["cpu_baseline"] = cpu_baseline(a.algo, a.dtype, c)
    if world == 1 and (a.sweep == "on" or (a.sweep == "auto" and a.workload == "cfg5")):
        out["sweep"] = sweep(c, st)


def per_kernel_times(algo, x, w, y, ws, st, nl, C, K, H, W, dt, reps, lay=0):
    import torch
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200._lib import lib, check, DTYPES
    import ctypes
    g = Wn.geometry(algo, nl, C, H, W, K, 1, dt)
    es = 4 if dt == "fp32" else 2
    U = ws.data_ptr()
    nbU = g["planes"] * g["S"] * K * g["Cp"] * es
    V = U + ((nbU + 1023) // 1024) * 1024
    nbV = g["planes"] * g["Q"] * g["T"] * g["Cp"] * es
    M = V + ((nbV + 1023) // 1024) * 1024
    L = lib()
    s = ctypes.c_void_p(st.cuda_stream)
    d = DTYPES[dt]
    calls = {
        "weight_transform": lambda: L.wino_weight_transform(ctypes.c_void_p(w.data_ptr()), K, C, algo.handle, d,
                                                            ctypes.c_void_p(U), s),
        "input_transform": lambda: L.wino_input_transform(ctypes.c_void_p(x.data_ptr()), nl, C, H, W, 1,
                                                          algo.handle, d, lay, ctypes.c_void_p(V), s),
        "domain_gemm": lambda: L.wino_domain_gemm(ctypes.c_void_p(V), ctypes.c_void_p(U), g["T"], C, K,
                                                  algo.handle, d, ctypes.c_void_p(M), s),
        "output_transform": lambda: L.wino_output_transform(ctypes.c_void_p(M), nl, K, H, W, 1, algo.handle, d, lay,
                                                            ctypes.c_void_p(y.data_ptr()), s),
    }
    names = list(calls)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(reps)]
    for _ in range(2):
        for n in names:
            check(calls[n]())
    torch.cuda.synchronize()
    for r in range(reps):
        evs[r][0].record(st)
        for i, n in enumerate(names):
            check(calls[n]())
            evs[r][i + 1].record(st)
    torch.cuda.synchronize()
    return {n: sum(evs[r][i].elapsed_time(evs[r][i + 1]) for r in range(reps)) / reps for i, n in enumerate(names)}


def e2e(algo, x, w, y, ws, st, nl, C, K, H, W, a, world, dist):
    import torch
    import paper_1905_05233_b200 as Wn
    xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
    steps = max(5, min(a.steps, 30))
    for _ in range(2):
        Wn.wino_conv2d_host_io(xh, x, w, algo, y, yh, ws, stream=st, layout=a.layout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        Wn.wino_conv2d_host_io(xh, x, w, algo, y, yh, ws, stream=st, layout=a.layout)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        from paper_1905_05233_b200 import distributed as D
        ms = D.max_over_ranks(ms, dist, "cuda")
    N = nl * world
    return {"value": direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": x.numel() * x.element_size() * world,
            "d2h_bytes_per_step": y.numel() * y.element_size() * world,
            "path": "wino_conv2d_host_io: pinned x -> device, layer, device y -> pinned host"}


def sweep(c, st):
    """Tile-size / polynomial-set sweep of cfg5 (BASELINE configs[4]) on one GPU."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    rows = []
    N, C, K, H, W = c["N"], c["C"], c["K"], c["H"], c["W"]
    for dt in ("bf16", "fp16", "fp32"):
        tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
        x64, w64 = datagen.layer(N, C, K, H, W, dt, seed=0, xdist=c["xdist"])
        x = torch.from_numpy(x64).to(tdt).cuda()
        w = torch.from_numpy(w64).to(tdt).cuda()
        del x64
        yref = Wn.wino_direct_conv2d_f64(x, w, 1, stream=st)
        for name in ("lin2", "sup1_2", "lin3", "lin4", "sup1_4", "lin6", "sup1_6", "lin8", "sup1_8"):
            spec, m = canonical_spec(name)
            algo = Wn.WinoAlgo(spec, m)
            y = torch.empty((N, K, H, W), dtype=tdt, device="cuda")
            ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, N, C, H, W, K, 1, dt))
            for _ in range(3):
                Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(10):
                Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            s = Wn.summary(Wn.wino_error_stats(y, yref, m, stream=st).cpu())
            rows.append({"algo": name, "dtype": dt, "mu": algo.mu, "ratio": round(algo.ratio_2d, 4), "ms": ms,
                         "tflops_direct_eq": direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12,
                         "rel_l1": s["rel_l1"], "mean_rel": s["mean_rel"], "nonfinite": s["nonfinite"]})
            del ws, y
        del x, w, yref
        torch.cuda.empty_cache()
    return rows


def ncu_traffic(kernel, a):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if one
    matches this workload (profiles/ncu_full_*.json), else None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_*.json"))):
        try:
            with open(p) as f:
                d = json.load(f)
            e = d.get(f"{a.workload}/{a.algo}/{a.dtype}/{kernel}")
            if e:
                return e.get("dram_bytes")
        except Exception:
            pass
    return None


if __name__ == "__main__":
    main()
