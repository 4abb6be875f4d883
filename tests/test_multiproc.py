"""N>1 host logic on CPU (gloo, world size 2): batch partitioning and the
reduction of the 8 error statistics.  The statistics of a
sharded run must equal those of one process over the whole batch: the oracle's
stats8 (oracle/metrics.py) is computed per rank slice and reduced with
paper_1905_05233_b200.distributed.reduce_stats."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
from oracle import conv as CV
from oracle import metrics as MT
from oracle import precision as P
from oracle import transforms as T
from paper_1905_05233_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    x, w = datagen.layer(4, 6, 5, 9, 11, "bf16", seed=3)
    mods, m = T.canonical("lin4")
    ts = T.make_transforms(mods, m)
    y = P.pipeline_conv2d(ts, x, w, "bf16")
    yref = CV.direct_conv2d_f64(x, w, 1)
    return x, w, y, yref, m


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, y, yref, m = _case()
        lo, hi = D.batch_slice(x.shape[0], world, rank)
        s = torch.tensor(MT.stats8(y[lo:hi], yref[lo:hi], m), dtype=torch.float64)
        s = D.reduce_stats(s, dist)
        t = D.max_over_ranks(1.0 + rank, dist, "cpu")
        if rank == 0:
            q.put((s.numpy().tolist(), t))
    finally:
        dist.destroy_process_group()


def test_batch_slice():
    assert [D.batch_slice(256, 8, r) for r in (0, 7)] == [(0, 32), (224, 256)]
    with pytest.raises(ValueError):
        D.batch_slice(10, 4, 0)


def test_sharded_stats_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, w, y, yref, m = _case()
    want = MT.stats8(y, yref, m)
    np.testing.assert_allclose(got, want, rtol=1e-12)
    assert tmax == 2.0


def test_reduce_stats_single_rank_identity():
    class _One:
        class ReduceOp:
            SUM, MAX = "sum", "max"

        @staticmethod
        def all_reduce(t, op=None, group=None):
            return None
    s = torch.arange(8, dtype=torch.float64)
    assert torch.equal(D.reduce_stats(s, _One), s)
