"""N>1 host logic of bench.py on CPU: the
self-launcher's torchrun command, the strong-scaling batch split, and -- under
a real torchrun with the gloo backend, world sizes 2 and 4 -- that the
per-rank statistics of the split batch reduce (distributed.reduce_stats) to
exactly the single-process statistics of the whole batch, so the error numbers
are identical for every GPU count.  The device step is stood in for by the
oracle's pipeline-mode emulation (this is a test of the host plumbing)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import bench
import datagen
from oracle import conv as CV
from oracle import metrics as MT
from oracle import precision as P
from oracle import transforms as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_launcher_cmd():
    cmd = bench.launcher_cmd(["--gpus", "8", "--steps", "20"], 8, 29511)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and "--master-port=29511" in cmd
    assert cmd[-5].endswith("bench.py") and cmd[-4:] == ["--gpus", "8", "--steps", "20"]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_batch_strong_partitions_the_global_batch(world):
    sl = [bench.rank_batch(256, world, r, "strong") for r in range(world)]
    assert sl[0][0] == 0 and sl[-1][1] == 256
    assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
    assert len({hi - lo for lo, hi in sl}) == 1
    assert all(bench.rank_batch(256, world, r, "weak") == (0, 256) for r in range(world))


WORKER = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
import bench, datagen
from oracle import conv as CV, metrics as MT, precision as P, transforms as T
from paper_1905_05233_b200 import distributed as D
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
N, C, K, H, W = 8, 6, 5, 9, 11
x, w = datagen.layer(N, C, K, H, W, "bf16", seed=0)        # the global batch, drawn once
lo, hi = bench.rank_batch(N, world, rank, "strong")
mods, m = T.canonical("lin4")
ts = T.make_transforms(mods, m)
y = P.pipeline_conv2d(ts, x[lo:hi], w, "bf16")               # stands in for the device step
yref = CV.direct_conv2d_f64(x[lo:hi], w, 1)
s = D.reduce_stats(torch.tensor(MT.stats8(y, yref, m), dtype=torch.float64), dist)
t = D.max_over_ranks(1.0 + rank, dist, "cpu")
if rank == 0:
    with open(sys.argv[2], "w") as f:
        json.dump({"stats": s.tolist(), "tmax": t, "world": world, "slice": [lo, hi]}, f)
dist.destroy_process_group()
"""


@pytest.mark.parametrize("world", [2, 4])
def test_torchrun_gloo_stats_identical_across_world_sizes(world, tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = tmp_path / "out.json"
    cmd = bench.launcher_cmd([ROOT, str(out)], world, _free_port(), script=str(script))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "1"
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(out.read_text())
    assert got["world"] == world and got["tmax"] == float(world) and got["slice"] == [0, 8 // world]
    x, w = datagen.layer(8, 6, 5, 9, 11, "bf16", seed=0)
    mods, m = T.canonical("lin4")
    ts = T.make_transforms(mods, m)
    want = MT.stats8(P.pipeline_conv2d(ts, x, w, "bf16"), CV.direct_conv2d_f64(x, w, 1), m)
    np.testing.assert_allclose(got["stats"], want, rtol=1e-12, atol=0)
