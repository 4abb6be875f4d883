"""Build libwino.so in-tree: nvcc for sm_100a (tcgen05 / TMA need the 'a'
target), -lineinfo for ncu source mapping, no --use_fast_math (subnormals and
round-to-nearest-even must be kept, readings A10/A11).

    python -m paper_1905_05233_b200.build [--force] [-j N]
"""
import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libwino.so")
# (source, object name, extra defines): xform.cu is compiled once per dtype x kind
# (input / output transform) x m-range slice, so its large instantiations build in parallel
XFORM = [("xform.cu", f"xform_{k}_{d}_{p}.cu", [f"-DWINO_XF_DT={d}", f"-DWINO_XF_KIND={k}", f"-DWINO_XF_PART={p}"])
         for k in (0, 1) for d in (0, 1, 2) for p in (0, 1, 2)]
UNITS = XFORM + [(s, s, []) for s in ["capi_host.cpp", "generator.cpp", "transforms.cu", "gemm.cu", "split.cu",
                                      "conv.cu", "misc.cu"]]
SOURCES = sorted({u[0] for u in UNITS})
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _flags(src):
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]
    if src.endswith(".cu"):
        return ARCH + common + ["-lineinfo", "-Xptxas", "-warn-spills"]
    return ["-x", "c++"] + common


def _deps(src):
    """src and the local headers it includes (transitively): an edit to one
    kernel file rebuilds only the objects that see it."""
    inc = [CSRC, os.path.join(HERE, "..", "include")]
    seen, todo = set(), [os.path.join(CSRC, src)]
    while todo:
        f = todo.pop()
        if f in seen:
            continue
        seen.add(f)
        with open(f) as fh:
            for line in fh:
                line = line.strip()
                if line.startswith("#include") and '"' in line:
                    name = line.split('"')[1]
                    for d in [os.path.dirname(f)] + inc:
                        c = os.path.normpath(os.path.join(d, name))
                        if os.path.exists(c):
                            todo.append(c)
                            break
    return sorted(seen)


def build(force=False, jobs=None, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    objs, todo = [], []
    # the largest units first (they bound the wall time)
    for s, name, defs in sorted(UNITS, key=lambda u: (u[0] != "xform.cu", u[2][1:] if u[2] else [])):
        o = os.path.join(OBJ, name + ".o")
        objs.append(o)
        dep_mtime = max(os.path.getmtime(p) for p in _deps(s))
        if force or not os.path.exists(o) or os.path.getmtime(o) < dep_mtime:
            todo.append((s, o, defs))

    def compile_one(item):
        s, o, defs = item
        cmd = [nvcc()] + _flags(s) + defs + ["-c", os.path.join(CSRC, s), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr)
        return os.path.basename(o)

    if todo:
        with ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 1)) as ex:
            for s in ex.map(compile_one, todo):
                if verbose:
                    print("compiled", s)
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    print(build(a.force, a.j, verbose=True))
    sys.exit(0)
