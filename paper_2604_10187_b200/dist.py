"""Multi-GPU decision grids and fits.  Grids: the flattened shape index (pair-major, M-minor)
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
    if staging.device.type == "cuda" and dist.get_backend(group) != "nccl":
        host = staging.cpu()  # gloo with device tensors: through the host
        dist.all_gather_into_tensor(host, host[rank * per: rank * per + per], group=group)
        staging.copy_(host)
    else:
        dist.all_gather_into_tensor(staging, mine, group=group)
    local_full.copy_(staging[:n_entries])
    return staging


def fused_sharded_sweep(grid, group=None, stream=None):
    """The sweep with the exchange fused into its epilogue: every rank maps
    its peers' grid storages (CUDA IPC over NVLink) and its sweep kernel
    stores each entry of its slice into all of them -- the transfer overlaps
    the computation tile by tile and no all-gather follows.  Two barriers:
    mappings ready, all stores landed; then each rank rebuilds its run index.
    (Single-process tests drive the same multi-destination epilogue with
    several local grids: tests/test_gpu_decide.py::test_sweep_to_*.)"""
    from . import capi

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = grid.engine.device
    lo, hi, _ = shard_bounds(grid.n_entries, world, rank)
    mine = grid.ipc_handle()
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    dests, opened = [grid.entries_ptr], []
    try:
        for r in range(world):
            if r != rank:
                ent, base = capi.ipc_open(handles[r][0], handles[r][1], dev)
                dests.append(ent)
                opened.append(base)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)
        if hi > lo:
            grid.sweep_to(dests, lo, hi, stream=stream)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)
        grid.finalize(stream=stream)
    finally:
        for b in opened:
            capi.ipc_close(b)
    return grid


def sharded_sweep(grid, group=None, stream=None):
    """Fill `grid` (a capi.Grid, identical on every rank) cooperatively:
    each rank sweeps its slice, then the NCCL all-gather replicates it.
    Everything is ordered on `stream` (default: the current stream)."""
    ent = grid.entries_tensor()
    st = stream if stream is not None else torch.cuda.current_stream(ent.device)

    def fill(lo, hi):
        grid.sweep(lo, hi, stream=st)

    with torch.cuda.stream(st):
        gather_grid(ent, grid.n_entries, group=group, fill=fill)
    grid.finalize(stream=st)
    return ent


# ---------------------------------------------------------------- sharded fit
# build_dual_table fits every macro from its own records only (model.cpp:194-
# 253: records grouped by macro, macros visited in registry order), so the
# fit shards by macro: each rank fits a contiguous slice of the registry and
# the per-rank table sets are concatenated in rank order, which is registry
# order.  W must be global: the reference takes params.W, or the largest
# record wave when W <= 0 -- an all-reduce(max) here.

_PER_TABLE = {"macro_id": 1, "theta_ext": 4, "ext_flags": 1, "W_arr": 1, "lin_theta": 4, "lin_r2": 1,
              "lin_mape": 1, "lin_degenerate": 1}
# CSR groups: offsets key -> (per-entry arrays with their widths)
_CSR = {
    "coeff_off": {"coeff_w": 1, "coeff_theta": 4, "diag_r2": 1, "diag_mape": 1, "diag_samples": 1, "diag_flags": 1},
    "ext_aoff": {"ext_l": 1, "ext_micro": 1},
    "step_off": {"step_l": 1, "step_t": 1},
}


def macro_shards(registry_ids, world: int):
    """Contiguous slices of the registry (registry order), one per rank."""
    import numpy as np

    ids = np.asarray(registry_ids)
    per = -(-len(ids) // world)
    return [ids[r * per: (r + 1) * per] for r in range(world)]


def records_of(records: dict, ids):
    """The records whose macro is in `ids` (order preserved)."""
    import numpy as np

    m = np.isin(records["macro"], ids)
    return {k: v[m] for k, v in records.items()}


def merge_tables(parts):
    """Concatenate table sets (fit_build outputs, in registry order) into one.
    Empty parts (n_tables == 0) are skipped."""
    import numpy as np

    parts = [p for p in parts if p and p["n_tables"] > 0]
    if not parts:
        raise RuntimeError("no tables built")
    out = {"n_tables": sum(p["n_tables"] for p in parts), "W": parts[0]["W"], "p": parts[0]["p"],
           "device_ms": max(p.get("device_ms", 0.0) for p in parts)}
    for k in _PER_TABLE:
        out[k] = np.concatenate([p[k] for p in parts])
    for off, members in _CSR.items():
        offs, base = [np.zeros(1, np.int32)], 0
        for p in parts:
            offs.append(p[off][1:] + base)
            base += int(p[off][-1])
        out[off] = np.concatenate(offs).astype(np.int32)
        for k in members:
            out[k] = np.concatenate([p[k] for p in parts])
    # anchors: awave_off over waves, awave_aoff over anchors
    aw, an = [np.zeros(1, np.int32)], [np.zeros(1, np.int32)]
    bw = ba = 0
    for p in parts:
        aw.append(p["awave_off"][1:] + bw)
        an.append(p["awave_aoff"][1:] + ba)
        bw += int(p["awave_off"][-1])
        ba += int(p["awave_aoff"][-1])
    out["awave_off"] = np.concatenate(aw).astype(np.int32)
    out["awave_aoff"] = np.concatenate(an).astype(np.int32)
    for k in ("awave_w", "anchor_l", "anchor_micro", "anchor_partial"):
        out[k] = np.concatenate([p[k] for p in parts])
    return out


def sharded_fit(records: dict, registry_ids, W: int = 0, p: int = 10, group=None, fit=None, device: int = 0):
    """build_dual_table sharded by macro over the ranks of `group`; every
    rank returns the full table set.  `fit(records, ids, W, p, device)`
    defaults to the GPU fit (capi.fit_build); the CPU tests pass a stand-in.
    The exchange is one all_gather_object of the per-rank tables (a few MB,
    NCCL over NVLink on B200)."""
    import numpy as np

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if fit is None:
        from . import capi

        fit = capi.fit_build
    if W <= 0:  # the reference's "max r.w over all records", made global
        wmax = torch.tensor([int(np.max(records["w"])) if len(records["w"]) else 0], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            wmax = wmax.cuda()
        dist.all_reduce(wmax, op=dist.ReduceOp.MAX, group=group)
        W = int(wmax.item())
    ids = macro_shards(registry_ids, world)[rank]
    mine = records_of(records, ids)
    part = fit(mine, ids, W, p, device) if len(ids) and len(mine["g"]) else None
    parts = [None] * world
    dist.all_gather_object(parts, part, group=group)
    return merge_tables(parts)


# ------------------------------------------------- device-resident sharded build
# The multi-GPU build keeps the tables on the devices end to end: each rank
# fits its registry slice from records resident in its HBM (wt_fit_build_
# device), packs the tables into one blob (wt_build_pack), ONE all-gather
# moves the blobs (NCCL over NVLink; equal strides, this rank's blob written
# in place at its slot), and every rank merges them into the full build on
# its device (wt_build_merge) and resolves its engine image there
# (Engine.from_build).  Host traffic: two tiny all-gathers of counts/sizes
# and the merged build's macro ids.

PACK_ALIGN = 256


def exchange_packed(nbytes: int, counts, pack, device, group=None):
    """All-gather variable-size packed blobs.  `pack(dst)` writes this rank's
    blob into the uint8 tensor `dst` (its slot of the gather buffer).
    Returns (buffer [world * stride] uint8, stride, counts [world, 5]).
    Ranks with nothing to send pass nbytes 0 and counts of zeros."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    meta_dev = device if nccl else "cpu"
    meta = torch.tensor([int(nbytes)] + [int(c) for c in counts], dtype=torch.int64, device=meta_dev)
    allm = torch.empty((world, 6), dtype=torch.int64, device=meta_dev)
    dist.all_gather_into_tensor(allm.view(-1), meta, group=group)
    allm = allm.cpu()
    stride = -(-int(allm[:, 0].max()) // PACK_ALIGN) * PACK_ALIGN
    stride = max(stride, PACK_ALIGN)
    buf = torch.empty(world * stride, dtype=torch.uint8, device=device)
    mine = buf[rank * stride: (rank + 1) * stride]
    if nbytes:
        pack(mine)
    if nccl:
        dist.all_gather_into_tensor(buf, mine, group=group)  # in place
    else:  # gloo (CPU tests; two processes on one GPU): staged through the host
        host = buf.cpu() if buf.device.type != "cpu" else buf
        dist.all_gather_into_tensor(host, host[rank * stride: (rank + 1) * stride], group=group)
        if host is not buf:
            buf.copy_(host)
    return buf, stride, allm[:, 1:].numpy()


def shard_records(records: dict, registry_ids, world: int, rank: int):
    """This rank's macro slice and the records of those macros (host arrays)."""
    ids = macro_shards(registry_ids, world)[rank]
    return ids, records_of(records, ids)


def sharded_build(records_dev: dict, shard_ids, W: int, p: int = 10, group=None, device: int = 0, stream=None):
    """build_dual_table sharded by macro, tables kept on the devices.
    `records_dev`: this rank's records (device tensors, capi.Build layout) of
    the macros `shard_ids` (its contiguous registry slice, macro_shards).
    W must be the global horizon (> 0; the reference's W <= 0 rule is a
    global max -- resolve it first with global_w).  Returns the merged
    capi.Build on this rank's device (the full registry's tables)."""
    from . import capi

    st = stream if stream is not None else torch.cuda.current_stream(device)
    if W <= 0:
        raise ValueError("sharded_build needs the global W (global_w)")
    part = None
    if len(shard_ids) and int(records_dev["g"].numel()):
        part = capi.Build(records_dev, shard_ids, W, p, device=device, stream=st)
    try:
        if part is not None:
            counts, nbytes = part.pack_info()
        else:
            counts, nbytes = [0, 0, 0, W, p], 0
        with torch.cuda.stream(st):
            buf, stride, allc = exchange_packed(nbytes, counts, lambda dst: part.pack(dst, stream=st),
                                                torch.device("cuda", device), group=group)
        return capi.Build.merge(buf, stride, allc, device=device, stream=st)
    finally:
        if part is not None:
            part.close()


def global_w(records_w, group=None, device=None):
    """The reference's W for params.W <= 0: max r.w over ALL records
    (model.cpp:201-203), an all-reduce(max) over the ranks' shards."""
    import numpy as np

    w = int(np.max(records_w)) if len(records_w) else 0
    t = torch.tensor([w], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.to(device if device is not None else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())
