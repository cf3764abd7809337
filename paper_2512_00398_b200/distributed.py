"""DM-trial sharding across the GPUs of one node.

One process per GPU.  Every rank searches the whole file for a contiguous block
of DM trials (blocks balanced by dedispersion work, sum over chunks of
(L - maxdelay_t) * nchans); trials are independent, so no data-path collective
is needed.  The single exchange step is the candidate gather: counts with an
all_gather, then the fixed-width 72-byte records padded to the largest count
(NCCL over NVLink for CUDA tensors, gloo for the CPU tests).  Rank 0 re-sorts by
(peak_sample, dm_trial, width_index) -- exactly the order a single device
produces -- and runs link_grid, so the output is identical for any world size.
"""
from __future__ import annotations

import numpy as np

from . import abi


def trial_work(plan, chunk_lengths) -> np.ndarray:
    """Channel-adds of each trial summed over the file's chunks."""
    maxd = plan.delays.max(axis=1).astype(np.int64)
    w = np.zeros(plan.ntrials, np.float64)
    for L in chunk_lengths:
        w += np.maximum(0, int(L) - maxd)
    return w * plan.nchans


DD_TRIAL_BLOCK = 32  # trials per dedispersion CTA (csrc: 16 warps x 2 trials)


def shard_trials(work: np.ndarray, world: int, granule: int = 1) -> list[tuple[int, int]]:
    """Contiguous trial ranges with (near-)equal total work; every range non-empty
    when ntrials >= world.

    granule > 1 (the dedispersion kernel's 32-trial block): ranges start on multiples of
    `granule` and a block costs `granule` x its longest trial's work -- a block with
    fewer trials takes as long as a full one, so a shard of 119 trials (3 full blocks
    + 23) would pay 7 % for the partial block."""
    n = len(work)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    if granule > 1 and n >= granule * world:
        nb = (n + granule - 1) // granule
        bcost = np.array([granule * work[b * granule:(b + 1) * granule].max() for b in range(nb)])
        inner = shard_trials(bcost, world, 1)
        return [(lo * granule, min(n, hi * granule)) for lo, hi in inner]
    cum = np.concatenate([[0.0], np.cumsum(work)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        b = min(max(b, bounds[-1] + (1 if n - bounds[-1] > world - r else 0)), n - (world - r))
        bounds.append(max(b, bounds[-1]))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def sort_candidates(c: np.ndarray) -> np.ndarray:
    """(peak_sample, dm_trial, width_index) order, src/pipeline.cpp:100-105."""
    if len(c) < 2:
        return c
    order = np.lexsort((c["width_index"], c["dm_trial"], c["peak_sample"]))
    return c[order]


def gather_candidates(local: np.ndarray, *, device=None, group=None) -> np.ndarray | None:
    """All ranks contribute their candidate records; rank 0 gets the merged, sorted list
    (other ranks get None).  Records travel as raw bytes in one padded all_gather."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    itemsize = abi.CANDIDATE_DTYPE.itemsize
    dev = device if device is not None else torch.device("cpu")
    n = torch.tensor([len(local)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(1, max(counts))
    buf = torch.zeros(cap * itemsize, dtype=torch.uint8, device=dev)
    if len(local):
        raw = torch.from_numpy(np.ascontiguousarray(local).view(np.uint8).copy())
        buf[: raw.numel()] = raw.to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    if rank != 0:
        return None
    # (np.concatenate would canonicalise the padded 72-byte record dtype)
    merged = np.zeros(sum(counts), abi.CANDIDATE_DTYPE)
    raw = merged.view(np.uint8)
    off = 0
    for r, b in enumerate(bufs):
        if counts[r]:
            nb = counts[r] * itemsize
            raw[off: off + nb] = b[:nb].cpu().numpy()
            off += nb
    return sort_candidates(merged)


def search_file_distributed(payload, task, *, rank: int, world: int, device: int, group=None):
    """Sharded file search; rank 0 returns the SearchResult, other ranks None."""
    import torch

    from .engine import default_engine
    from .pipeline import SearchResult

    work = trial_work(task.plan, [c.length for c in task.chunks])
    lo, hi = shard_trials(work, world, DD_TRIAL_BLOCK)[rank]
    eng = default_engine(device)
    cands, _, skipped = eng.search_file(payload, task.header.nsamples, task.chunks, task.plan,
                                        task.engine, trial_range=(lo, hi), cluster=False)
    merged = gather_candidates(cands, device=torch.device("cuda", device), group=group)
    if rank != 0:
        return None
    clusters = eng.link_grid(merged, task.engine.radii)
    return SearchResult(merged, clusters, skipped)
