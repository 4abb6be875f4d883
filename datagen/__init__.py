"""Seeded synthetic inputs shared by the oracle side and the GPU side.

Holds NO arithmetic of the method: it only draws random numbers and rounds them
to the storage dtype with library casts (numpy / torch CPU), which is how the
inputs of the paper's workloads are stood in for (DESIGN.md
"Input recipe").  numpy ``default_rng(seed)`` (PCG64); x is drawn first, then w,
in fp64, then rounded to the dtype (RNE).  The GPU receives exactly these bits.
"""
import numpy as np

DTYPES = ("fp32", "fp16", "bf16")


def to_dtype_values(a64, dtype):
    """Round an fp64 array to the dtype (library casts) and return the values as
    fp64 (exact: every dtype value is an fp64 value)."""
    a64 = np.asarray(a64, np.float64)
    if dtype == "fp64":
        return a64
    if dtype == "fp32":
        return a64.astype(np.float32).astype(np.float64)
    if dtype == "fp16":
        return a64.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        import torch
        return torch.from_numpy(a64).to(torch.bfloat16).to(torch.float64).numpy()
    raise ValueError(dtype)


def he_sigma(C, r=3):
    """He-normal std sqrt(2 / (r*r*C_in))."""
    return float(np.sqrt(2.0 / (r * r * C)))


def draw(rng, shape, dist):
    if dist == "uniform01":
        return rng.random(shape)
    if dist == "relu_normal":
        return np.maximum(0.0, rng.standard_normal(shape))
    if dist.startswith("normal:"):
        return rng.normal(0.0, float(dist.split(":")[1]), shape)
    if dist == "paper_trunc_normal":           # N(0, 1/3) rejected outside (-1, 1)
        out = rng.normal(0.0, 1.0 / 3.0, shape)
        bad = np.abs(out) >= 1
        while bad.any():
            out[bad] = rng.normal(0.0, 1.0 / 3.0, int(bad.sum()))
            bad = np.abs(out) >= 1
        return out
    raise ValueError(dist)


def layer(N, C, K, H, W, dtype, seed=0, xdist="relu_normal", wdist="he", r=3):
    """(x[N,C,H,W], w[K,C,r,r]) as fp64 arrays of dtype values."""
    rng = np.random.default_rng(seed)
    x = draw(rng, (N, C, H, W), xdist)
    wd = f"normal:{he_sigma(C, r)}" if wdist == "he" else wdist
    w = draw(rng, (K, C, r, r), wd)
    return to_dtype_values(x, dtype), to_dtype_values(w, dtype)


def tiles1d(T, n, dtype, seed=0, r=3):
    """BASELINE cfg 2: x[T, n+2] ~ U[0,1), h[T, 3] ~ N(0, 0.3)."""
    rng = np.random.default_rng(seed)
    x = rng.random((T, n + r - 1))
    h = rng.normal(0.0, 0.3, (T, r))
    return to_dtype_values(x, dtype), to_dtype_values(h, dtype)


# Named workloads (BASELINE.json configs).
CONFIGS = {
    "cfg1": dict(N=1, C=8, K=8, H=16, W=16, xdist="uniform01", dtype="fp32"),
    "cfg3": dict(N=32, C=256, K=256, H=56, W=56, xdist="relu_normal", dtype="fp16"),
    "cfg5": dict(N=256, C=512, K=512, H=28, W=28, xdist="relu_normal", dtype="bf16"),
}

VGG16 = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56),
         (256, 256, 56), (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28),
         (512, 512, 14), (512, 512, 14), (512, 512, 14)]
