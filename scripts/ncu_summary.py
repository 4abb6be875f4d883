"""Summarise ncu captures (run HERE, no GPU) into profiles/.

    python scripts/ncu_summary.py --tag r01 --key cfg5/lin4/bf16 \
        gpurun_out/prof_input_transform.ncu-rep ... [--launches gpurun_out/launches_r01.csv]

Writes profiles/ncu_full_<tag>.json ({"<key>/<kernel>": {metric: value}}, with
dram_bytes = dram__bytes_read.sum + dram__bytes_write.sum per launch; bench.py
reads it for roofline.traffic) and profiles/launches_<tag>.json (per-kernel
mean duration and share of the step from the --metrics gpu__time_duration.sum
launch list)."""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": "tc_inst_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_peak",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct_peak",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3}


def raw(rep):
    """Metrics of every kernel in an .ncu-rep, or in its `--page raw --csv` export (.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for i, n in enumerate(hdr):
            if n in METRICS:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if n.startswith("dram__bytes"):
                    v *= SCALE.get(u, 1)
                elif n == "gpu__time_duration.sum":
                    v *= SCALE.get(u, 1)   # -> us
                d[METRICS[n]] = v
        d["dram_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        res.append(d)
    return res


def short(name):
    for k in ("weight_transform", "input_transform", "domain_gemm", "output_transform", "conv1d_tiles",
              "stats", "direct_f64"):
        if k in name:
            return k
    return re.sub(r"[<(].*", "", name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--key", required=True, help="workload/algo/dtype")
    ap.add_argument("--launches")
    ap.add_argument("reps", nargs="*")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.reps:
        summ = {}
        p = os.path.join(ROOT, "profiles", f"ncu_full_{a.tag}.json")
        if os.path.exists(p):
            summ = json.load(open(p))
        for rep in a.reps:
            for d in raw(rep):
                d["source"] = os.path.basename(rep)
                summ[f"{a.key}/{short(d['kernel'])}"] = d
        json.dump(summ, open(p, "w"), indent=1, sort_keys=True)
        print("wrote", p)
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = {}
        for r in rows[1:]:
            k = short(r[ki])
            v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
            agg.setdefault(k, []).append(v)
        tot = sum(sum(v) for v in agg.values())
        out = {"key": a.key, "source": os.path.basename(a.launches),
               "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised launches; "
                       "compare shares, not absolutes",
               "kernels": {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot}
                           for k, v in agg.items()}}
        p = os.path.join(ROOT, "profiles", f"launches_{a.tag}.json")
        json.dump(out, open(p, "w"), indent=1)
        print("wrote", p)


if __name__ == "__main__":
    sys.exit(main())
