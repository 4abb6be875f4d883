#!/usr/bin/env python
"""Benchmark of the hot path: one step = one 2D Winograd conv layer through
libwino's C ABI (K2 weight transform, K1 input transform, K3 tcgen05
Winograd-domain GEMM, K4 output transform) over one batch of synthetic input.

Default workload (BASELINE.json configs[4], the largest single-GPU config the
metric is quoted on): N=256, C=K=512, 28x28, pad 1, post-ReLU inputs, He
weights; F(4x4, 3x3) Toom-Cook {0,-1,1,-1/2,1/2,inf} in bf16.  With --gpus N
(N > 1) the script re-launches itself under torchrun as N ranks, one per GPU
(NCCL); the global batch of 256 images is drawn once and split over the ranks
(strong scaling: the layer partitions over the batch with no exchange step,
DESIGN.md 8; --scaling weak gives every rank the whole batch).  The only
collective is the NCCL all-reduce of the error statistics, outside the timed
region.  Each rank's step is captured as one CUDA graph (--graph off: eager).

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
    ap.add_argument("--no-dtypes", action="store_true", help="skip the per-dtype roofline legs")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the workload's global batch is split over the ranks; weak: every rank runs it")
    ap.add_argument("--graph", default="on", choices=["on", "off"], help="time the step as one CUDA graph")
    ap.add_argument("--m-store", default="fp32", choices=["fp32", "dtype"],
                    help="M between K3 and K4: fp32 (reading R1) or rounded once to the layer dtype (reading M3)")
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
        "scaling": a.scaling, "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
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


# --------------------------------------------------------------------------- launcher


def launcher_cmd(argv, gpus, port, script=None):
    """torchrun command that re-runs this script (or `script`) as `gpus` ranks
    (one process per GPU, NCCL; rendezvous on 127.0.0.1).  Used when
    `--gpus N > 1` is given without a torchrun environment."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", script or os.path.abspath(__file__)] + list(argv)


def self_launch(a):
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    return subprocess.call(launcher_cmd(sys.argv[1:], a.gpus, port))


def rank_batch(n_global, world, rank, scaling):
    """Images [lo, hi) of the globally generated batch this rank runs.  Strong
    scaling (default): the global batch of the workload is split evenly over the
    ranks (paper_1905_05233_b200.distributed.batch_slice).  Weak scaling: every
    rank runs the whole workload batch (the same images, so the statistics stay
    comparable across rank counts)."""
    from paper_1905_05233_b200 import distributed as D
    if scaling == "weak":
        return 0, n_global
    return D.batch_slice(n_global, world, rank)


# --------------------------------------------------------------------------- our arm


def tc_peak_tflops(dtype, peaks):
    """Tensor peak for the dtype's contraction: bf16/fp16 = the measured bf16
    figure; fp32 runs three TF32 products, TF32 = bf16 x 1/2 (the guide's nominal
    dense ratio, 1.125 vs 2.25 PFLOP/s), so the fp32-accurate peak is bf16 / 6."""
    b = peaks["bf16_tflops"]
    return {"bf16": b, "fp16": b, "fp32": b / 2.0 / 3.0}[dtype]


def main():
    a = parse()
    if a.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(a, rank, world)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    if a.m_store == "dtype":
        algo.set_m_storage("dtype")
    tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[a.dtype]
    N = c["N"]                                      # the workload's (global) batch
    lo, hi = rank_batch(N, world, rank, a.scaling)
    nl = hi - lo                                    # images on this rank
    n_job = nl * world                              # images processed by the whole job per step
    # the global batch is drawn once from seed 0 (x first, then w); each rank keeps its slice
    x64, w64 = datagen.layer(N, c["C"], c["K"], c["H"], c["W"], a.dtype, seed=0, xdist=c["xdist"])
    x = torch.from_numpy(np.ascontiguousarray(x64[lo:hi])).to(tdt).cuda()
    if a.layout == "nhwc":
        x = x.permute(0, 2, 3, 1).contiguous()
    w = torch.from_numpy(w64).to(tdt).cuda()
    del x64
    C, K, H, W = c["C"], c["K"], c["H"], c["W"]
    Ho, Wo = H, W
    y = torch.empty((nl, K, Ho, Wo) if a.layout == "nchw" else (nl, Ho, Wo, K), dtype=tdt, device="cuda")
    ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, nl, C, H, W, K, 1, a.dtype, a.layout))
    st = torch.cuda.Stream()          # a side stream (graph capture needs one), current for the whole run
    torch.cuda.set_stream(st)

    def step():
        Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st, layout=a.layout)
        return Wn.wino_last_launch_count()

    with torch.cuda.stream(st):
        for _ in range(max(3, a.warmup)):
            per_step = step()
    torch.cuda.synchronize()
    graph = None
    if a.graph == "on":
        # the whole step (K2 fork/join on the library's side stream, K1, K3, K4) as one CUDA graph
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                per_step = step()
            torch.cuda.synchronize()
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 -- reported, then the eager loop is timed
            graph = None
            graph_err = f"{type(e).__name__}: {e}"[:200]

    def timed(steps, use_graph):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(steps):
                if use_graph:
                    graph.replay()
                else:
                    step()
            e1.record(st)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = e0.elapsed_time(e1) / steps
        if world > 1:
            from paper_1905_05233_b200 import distributed as D
            t = D.max_over_ranks(t, dist, "cuda")
        return t

    with ClockSampler(local) as clk:
        ms = timed(a.steps, graph is not None)
    launches = per_step * a.steps
    flops = direct_flops(n_job, C, K, Ho, Wo)
    value = flops / (ms * 1e-3) / 1e12

    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
           "warmup": max(3, a.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": a.scaling,
           "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
           "config": {"workload": c["desc"], "algo": f"{a.algo} {{{spec}}} m={m} mu={algo.mu} ratio={algo.ratio_2d:.4g}",
                      "lowering": a.lowering, "layout": a.layout, "m_store": a.m_store,
                      "global_batch": n_job, "per_gpu_batch": nl,
                      "parallelism": f"dp{world} (batch-partitioned, no data-path collective)",
                      "launch": "CUDA graph per step" if graph is not None else "eager",
                      "l2": "inputs larger than L2 (x %.0f MB per GPU; V and M staged through HBM)" % (
                          x.numel() * x.element_size() / 1e6)},
           "gpu_launches": launches, "clocks": clk.summary()}
    if a.graph == "on" and graph is None:
        out["config"]["graph_error"] = graph_err
    if not a.no_extras:
        out["ms_per_step_eager"] = timed(a.steps, False) if graph is not None else ms
        extras(a, out, algo, x, w, y, ws, st, nl, C, K, H, W, m, world, rank, dist, c, spec, graph, timed)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def layer_bytes(nl, C, K, H, W, es, g):
    """Compulsory (x + w + y) and staged (+ U, V and M written and read) bytes of
    one layer on one GPU; M is fp32 (R1) or 16-bit (M3)."""
    pl = g["planes"]
    xb, yb, wb = nl * C * H * W * es, nl * K * H * W * es, K * C * 9 * es
    Ub = pl * g["S"] * K * g["Cp"] * es
    Vb = pl * g["Q"] * g["T"] * g["Cp"] * es
    Mb = g["Q"] * K * g["T"] * g.get("mes", 4)
    return dict(x=xb, y=yb, w=wb, U=Ub, V=Vb, M=Mb, compulsory=xb + yb + wb, staged=xb + yb + wb + Ub + 2 * Vb + 2 * Mb)


def kernel_rooflines(algo, dtype, x, w, y, ws, st, nl, C, K, H, W, reps, lay, peaks, peak_src, a):
    """Per-kernel CUDA-event times and the roofline of the dominant kernel."""
    import paper_1905_05233_b200 as Wn
    g = Wn.geometry(algo, nl, C, H, W, K, 1, dtype)
    es = 4 if dtype == "fp32" else 2
    B = layer_bytes(nl, C, K, H, W, es, g)
    gemm_flops = 2.0 * g["T"] * C * K * g["S"] * (3 if dtype == "fp32" else 1)   # fp32: 3 TF32 products
    kern = per_kernel_times(algo, x, w, y, ws, st, nl, C, K, H, W, dtype, reps, lay=lay)
    hbm = peaks["hbm_gbs"] * 1e9
    tc = tc_peak_tflops(dtype, peaks) * 1e12 * (3 if dtype == "fp32" else 1)      # raw TF32 rate for fp32
    info = {
        "weight_transform": {"bytes": B["w"] + B["U"], "flops": None},
        "input_transform": {"bytes": B["x"] + B["V"], "flops": None},
        "domain_gemm": {"bytes": B["V"] + B["U"] + B["M"], "flops": gemm_flops},
        "output_transform": {"bytes": B["M"] + B["y"], "flops": None},
    }
    kernels = {}
    for k_, ms_ in kern.items():
        d = info[k_]
        t_mem = d["bytes"] / hbm
        t_tc = d["flops"] / tc if d["flops"] else 0.0
        kernels[k_] = {"us": ms_ * 1e3, "algorithmic_bytes": d["bytes"], "GB/s": d["bytes"] / (ms_ * 1e-3) / 1e9,
                       "TFLOP/s": (d["flops"] / (ms_ * 1e-3) / 1e12) if d["flops"] else None,
                       "bound": "tensor" if t_tc > t_mem else "hbm", "frac": max(t_mem, t_tc) / (ms_ * 1e-3)}
    dom = max(kernels, key=lambda k_: kernels[k_]["us"])
    mkey = dtype + ("_m3" if g.get("mes", 4) == 2 else "")   # ncu summary key of this M storage
    kd = kernels[dom]
    if kd["bound"] == "tensor":
        ach = info[dom]["flops"] / (kd["us"] * 1e-6) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": tc / 1e12, "unit": "TFLOP/s",
                "frac": ach / (tc / 1e12), "traffic": ncu_traffic(dom, a, mkey), "peak_source": peak_src}
    else:
        ach = info[dom]["bytes"] / (kd["us"] * 1e-6) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": ncu_traffic(dom, a, mkey), "peak_source": peak_src}
    if dtype == "fp32":
        roof["tf32_peak_note"] = ("3xTF32 (hi*hi + hi*lo + lo*hi); TF32 dense peak = measured bf16 %.1f TFLOP/s x 1/2 "
                                  "(nominal ratio 1.125/2.25 PFLOP/s); fp32-accurate peak = that / 3" % peaks["bf16_tflops"])
    return kernels, roof, B, gemm_flops


def layer_fracs(ms, B, gemm_flops, dtype, peaks, sustained=False):
    """North-star layer rooflines: compulsory bytes (the fused ideal) and staged
    bytes (this K1 -> K3 -> K4 design) against the dtype's tensor peak."""
    hbm = peaks["hbm_gbs"] * 1e9
    tcp = tc_peak_tflops(dtype, peaks) * 1e12
    if sustained:
        tcp *= peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) / peaks["bf16_tflops"]
    f = gemm_flops / (3 if dtype == "fp32" else 1)                  # fp32-accurate flops at the fp32-accurate peak
    t_roof = max(f / tcp, B["compulsory"] / hbm)
    t_staged = max(f / tcp, B["staged"] / hbm)
    return {"t_roof_us": t_roof * 1e6, "frac_compulsory": t_roof / (ms * 1e-3), "t_staged_us": t_staged * 1e6,
            "frac_staged": t_staged / (ms * 1e-3), "tensor_peak_tflops": tcp / 1e12}


def extras(a, out, algo, x, w, y, ws, st, nl, C, K, H, W, m, world, rank, dist, c, spec, graph, timed):
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
    s = stats.cpu()
    out["accuracy"] = {k: (float(v) if not isinstance(v, int) else v) for k, v in Wn.summary(s).items()}
    out["accuracy"]["stats8"] = [float(v) for v in s.tolist()]
    del yref
    # ---------------------------------------------------------------- per-kernel breakdown + roofline
    lay = 0 if a.layout == "nchw" else 1
    kernels, roof, B, gemm_flops = kernel_rooflines(algo, a.dtype, x, w, y, ws, st, nl, C, K, H, W,
                                                    max(20, a.steps // 4), lay, peaks, peak_src, a)
    out["kernels"] = kernels
    out["roofline"] = roof
    ms = out["ms_per_step"]
    out["layer_roofline"] = dict(layer_fracs(ms, B, gemm_flops, a.dtype, peaks), peaks=peak_src)
    # ---------------------------------------------------------------- sustained (long loop, power cap)
    if world == 1 and graph is not None:
        steps_s = max(200, int(2000.0 / max(ms, 1e-3)))   # ~2 s of back-to-back steps
        ms_s = timed(steps_s, True)
        out["sustained"] = {"steps": steps_s, "ms_per_step": ms_s,
                            "value": direct_flops(nl, C, K, H, W) / (ms_s * 1e-3) / 1e12,
                            "layer_roofline": layer_fracs(ms_s, B, gemm_flops, a.dtype, peaks, sustained=True)}
    # ---------------------------------------------------------------- the other dtypes (same workload, rank 0 slice)
    if world == 1 and a.workload == "cfg5" and not a.no_dtypes:
        out["rooflines_by_dtype"] = {a.dtype: {"roofline": roof, "layer_roofline": out["layer_roofline"],
                                               "ms_per_step": ms}}
        for dt in ("bf16", "fp16", "fp32"):
            if dt != a.dtype:
                out["rooflines_by_dtype"][dt] = dtype_roofline(a, algo, dt, c, st, peaks, peak_src)
        # the same layer with M stored in the 16-bit dtype (reading M3), bf16 and fp16
        if a.m_store == "fp32":
            from paper_1905_05233_b200.algos import canonical_spec as _cs
            sp_, m_ = _cs(a.algo)
            a16 = Wn.WinoAlgo(sp_, m_, lowering=a.lowering).set_m_storage("dtype")
            out["m_store_dtype"] = {dt: dtype_roofline(a, a16, dt, c, st, peaks, peak_src, accuracy=True)
                                    for dt in ("bf16", "fp16")}
    # ---------------------------------------------------------------- end to end (host buffers)
    out["e2e"] = e2e(algo, x, w, y, ws, st, nl, C, K, H, W, a, world, dist)
    # ---------------------------------------------------------------- CPU baseline (rank 0, N=1 only)
    if world == 1:
        out["cpu_baseline"] = cpu_baseline(a.algo, a.dtype, c)
    if world == 1 and (a.sweep == "on" or (a.sweep == "auto" and a.workload == "cfg5")):
        out["sweep"] = sweep(c, st, peaks)


def dtype_roofline(a, algo, dt, c, st, peaks, peak_src, accuracy=False):
    """Step time, dominant-kernel roofline and layer fractions of the workload in
    another dtype (same algorithm); accuracy=True adds the error statistics
    against the fp64 direct convolution (device)."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
    N, C, K, H, W = c["N"], c["C"], c["K"], c["H"], c["W"]
    x64, w64 = datagen.layer(N, C, K, H, W, dt, seed=0, xdist=c["xdist"])
    x = torch.from_numpy(x64).to(tdt).cuda()
    w = torch.from_numpy(w64).to(tdt).cuda()
    del x64
    y = torch.empty((N, K, H, W), dtype=tdt, device="cuda")
    ws = Wn.alloc_workspace(Wn.wino_conv2d_workspace(algo, N, C, H, W, K, 1, dt))
    with torch.cuda.stream(st):
        for _ in range(3):
            Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            Wn.wino_conv2d(x, w, algo, out=y, workspace=ws, stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    acc = None
    if accuracy:
        yref = Wn.wino_direct_conv2d_f64(x, w, 1, stream=st)
        s8 = Wn.wino_error_stats(y, yref, algo.m, stream=st).cpu()
        acc = {k: (float(v) if not isinstance(v, int) else v) for k, v in Wn.summary(s8).items()}
        del yref
    kernels, roof, B, gemm_flops = kernel_rooflines(algo, dt, x, w, y, ws, st, N, C, K, H, W, 20, 0, peaks,
                                                    peak_src, a)
    del x, w, y, ws
    torch.cuda.empty_cache()
    r = {"ms_per_step": ms, "value": direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12, "kernels": kernels,
         "roofline": roof, "layer_roofline": layer_fracs(ms, B, gemm_flops, dt, peaks)}
    if acc is not None:
        r["accuracy"] = acc
        r["m_store"] = getattr(algo, "m_store", "fp32")
    return r


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
    nbV = g["planes"] * g["Q"] * g["TB"] * 128 * g["Cp"] * es   # V is padded to whole 128-tile blocks
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
    with torch.cuda.stream(st):
        for _ in range(2):
            Wn.wino_conv2d_host_io(xh, x, w, algo, y, yh, ws, stream=st, layout=a.layout)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
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


def sweep(c, st, peaks):
    """Tile-size / polynomial-set sweep of cfg5 (BASELINE configs[4]) on one GPU,
    m = 2..8 with linear (Toom-Cook) and one-quadratic (a^2+1) sets, 16-bit dtypes
    with M in fp32 (R1) and in the dtype (M3); each row carries its own layer
    roofline fractions."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_05233_b200 as Wn
    from paper_1905_05233_b200.algos import canonical_spec
    rows = []
    N, C, K, H, W = c["N"], c["C"], c["K"], c["H"], c["W"]
    for dt, ms_ in (("bf16", "fp32"), ("bf16", "dtype"), ("fp16", "fp32"), ("fp16", "dtype"), ("fp32", "fp32")):
        tdt = {"fp32": torch.float32, "fp16": torch.float16, "bf16": torch.bfloat16}[dt]
        x64, w64 = datagen.layer(N, C, K, H, W, dt, seed=0, xdist=c["xdist"])
        x = torch.from_numpy(x64).to(tdt).cuda()
        w = torch.from_numpy(w64).to(tdt).cuda()
        del x64
        yref = Wn.wino_direct_conv2d_f64(x, w, 1, stream=st)
        for name in ("lin2", "sup1_2", "lin3", "sup1_3", "lin4", "sup1_4", "lin5", "sup1_5", "lin6", "sup1_6", "lin7",
                     "sup1_7", "lin8", "sup1_8"):
            spec, m = canonical_spec(name)
            algo = Wn.WinoAlgo(spec, m)
            if ms_ == "dtype":
                algo.set_m_storage("dtype")
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
            g = Wn.geometry(algo, N, C, H, W, K, 1, dt)
            B = layer_bytes(N, C, K, H, W, 4 if dt == "fp32" else 2, g)
            fr = layer_fracs(ms, B, 2.0 * g["T"] * C * K * g["S"] * (3 if dt == "fp32" else 1), dt, peaks)
            rows.append({"algo": name, "dtype": dt, "m_store": ms_ if (dt != "fp32" and m <= 8) else "fp32",
                         "mu": algo.mu, "ratio": round(algo.ratio_2d, 4), "ms": ms,
                         "tflops_direct_eq": direct_flops(N, C, K, H, W) / (ms * 1e-3) / 1e12,
                         "frac_compulsory": fr["frac_compulsory"], "frac_staged": fr["frac_staged"],
                         "rel_l1": s["rel_l1"], "mean_rel": s["mean_rel"], "nonfinite": s["nonfinite"]})
            del ws, y
        del x, w, yref
        torch.cuda.empty_cache()
    return rows


def ncu_traffic(kernel, a, dtype=None):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if one
    matches this workload (profiles/ncu_full_*.json), else None."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_*.json")), reverse=True):   # newest tag first
        try:
            with open(p) as f:
                d = json.load(f)
            e = d.get(f"{a.workload}/{a.algo}/{dtype or a.dtype}/{kernel}")
            if e:
                return e.get("dram_bytes")
        except Exception:
            pass
    return None


if __name__ == "__main__":
    main()
