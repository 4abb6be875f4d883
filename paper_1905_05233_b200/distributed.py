"""Multi-GPU plumbing of the hot path: the layer partitions
over the batch with no exchange step, so ranks run independent images and the
only collective is the reduction of the 8 error statistics (include/wino.h,
wino_error_stats) -- sums for entries 0-3 and 5-7, a max for entry 4 --
outside the timed region.  One process per GPU (torchrun), NCCL on B200,
gloo for the CPU tests; torch.distributed is plumbing only."""
import torch

MAX_ENTRY = 4   # stats[4] = max_t relative error; every other entry is a sum


def batch_slice(n_global, world, rank):
    """Images [lo, hi) of rank `rank` when a global batch is split evenly."""
    if n_global % world:
        raise ValueError(f"global batch {n_global} does not divide over {world} ranks")
    per = n_global // world
    return rank * per, (rank + 1) * per


def reduce_stats(stats, dist, group=None):
    """All-reduce an 8-entry fp64 stats tensor across ranks: sum, except the
    per-tile max relative error (entry 4), which is a max.  Returns a new tensor."""
    if stats.numel() != 8 or stats.dtype != torch.float64:
        raise ValueError("stats must be 8 fp64 values")
    s_sum = stats.clone()
    s_sum[MAX_ENTRY] = 0
    dist.all_reduce(s_sum, op=dist.ReduceOp.SUM, group=group)
    s_max = stats[MAX_ENTRY:MAX_ENTRY + 1].clone()
    dist.all_reduce(s_max, op=dist.ReduceOp.MAX, group=group)
    s_sum[MAX_ENTRY] = s_max[0]
    return s_sum


def max_over_ranks(value, dist, device, group=None):
    """The slowest rank's time (the bench's timing rule)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
