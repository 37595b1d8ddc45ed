"""Multi-GPU decision grids: the flattened shape index (pair-major, M-minor)
is cut into equal contiguous slices, one per rank; every rank sweeps its
slice into its own grid (wt_sweep over [begin, end)), then one NCCL
all-gather over NVLink assembles the full grid on every rank.  The sweep is
embarrassingly parallel (every shape costs the same C evaluations), so the
static split is balanced; the all-gather is the only exchange.

torch.distributed is the plumbing: one process per GPU, backend "nccl" on
B200 (gloo in the CPU tests, where `fill` stands in for the device sweep).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ENTRY_INTS = 8  # wt_grid_entry is 32 bytes = 8 x int32


def shard_bounds(n_entries: int, world: int, rank: int):
    """Equal slices of ceil(n / world) entries; the last may be short."""
    per = -(-n_entries // world)
    lo = min(n_entries, rank * per)
    hi = min(n_entries, lo + per)
    return lo, hi, per


def gather_grid(local_full: torch.Tensor, n_entries: int, group=None, fill=None):
    """`local_full` is this rank's [n_entries, 8] int32 grid storage (device
    view of wt_grid_entry).  `fill(lo, hi)` writes rows [lo, hi) into it (the
    rank's slice).  Returns the padded staging buffer after the all-gather;
    the full grid is copied back into `local_full`."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi, per = shard_bounds(n_entries, world, rank)
    if fill is not None and hi > lo:
        fill(lo, hi)
    staging = torch.empty((per * world, ENTRY_INTS), dtype=torch.int32, device=local_full.device)
    mine = staging[rank * per: rank * per + per]
    if hi > lo:
        mine[: hi - lo].copy_(local_full[lo:hi])
    # in-place all-gather: this rank's chunk already sits at its offset
    dist.all_gather_into_tensor(staging, mine, group=group)
    local_full.copy_(staging[:n_entries])
    return staging


def sharded_sweep(grid, group=None, stream=None):
    """Fill `grid` (a capi.Grid, identical on every rank) cooperatively:
    each rank sweeps its slice, then the NCCL all-gather replicates it."""
    ent = grid.entries_tensor()

    def fill(lo, hi):
        grid.sweep(lo, hi, stream=stream)

    gather_grid(ent, grid.n_entries, group=group, fill=fill)
    grid.finalize(stream=stream)
    return ent
