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

import ctypes

import numpy as np

from . import abi
from ._native import check, lib


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


def gather_records(local: np.ndarray, *, device=None, group=None) -> np.ndarray | None:
    """Concatenate every rank's fixed-width records on rank 0 (other ranks get None).
    Counts travel in one all_gather, then the raw bytes padded to the largest count in a
    second (NCCL over NVLink for CUDA devices, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    local = np.ascontiguousarray(local)
    itemsize = local.dtype.itemsize
    dev = device if device is not None else torch.device("cpu")
    n = torch.tensor([len(local)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(1, max(counts))
    buf = torch.zeros(cap * itemsize, dtype=torch.uint8, device=dev)
    if len(local):
        raw = torch.from_numpy(local.view(np.uint8).reshape(-1).copy())
        buf[: raw.numel()] = raw.to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    if rank != 0:
        return None
    # (np.concatenate would canonicalise the padded 72-byte record dtype)
    merged = np.zeros(sum(counts), local.dtype)
    raw = merged.view(np.uint8).reshape(-1)
    off = 0
    for r, b in enumerate(bufs):
        if counts[r]:
            nb = counts[r] * itemsize
            raw[off: off + nb] = b[:nb].cpu().numpy()
            off += nb
    return merged


def gather_candidates(local: np.ndarray, *, device=None, group=None) -> np.ndarray | None:
    """All ranks contribute their candidate records; rank 0 gets the merged list sorted
    by (peak_sample, dm_trial, width_index) -- the single-device order."""
    merged = gather_records(np.ascontiguousarray(local, abi.CANDIDATE_DTYPE), device=device, group=group)
    return None if merged is None else sort_candidates(merged)


def gather_skipped(pairs: np.ndarray, *, device=None, group=None) -> np.ndarray | None:
    """(chunk, trial) skipped pairs of every shard, merged on rank 0 and sorted by
    (chunk, trial) -- FileOutcome::skipped_trials order (src/pipeline.cpp:95-96)."""
    pairs = np.ascontiguousarray(np.asarray(pairs, np.uint64).reshape(-1, 2))
    rec = pairs.view(np.dtype([("chunk", "<u8"), ("trial", "<u8")])).reshape(-1)
    merged = gather_records(rec, device=device, group=group)
    if merged is None:
        return None
    merged = np.sort(merged, order=("chunk", "trial"))
    return merged.view(np.uint64).reshape(-1, 2)


def row_slices(nsamples: int, world: int) -> list[tuple[int, int]]:
    """Rows of the file each rank uploads from host memory (equal contiguous slices)."""
    return [(nsamples * r // world, nsamples * (r + 1) // world) for r in range(world)]


class PayloadFanout:
    """Multi-GPU input path: every rank uploads 1/N of the file's rows from host memory
    into its own device buffer, then pulls the other ranks' rows over NVLink from their
    buffers (CUDA IPC, cudaMemcpyAsync between peers).  The host link carries each byte
    once per node instead of once per GPU; NCCL stays reserved for the candidate gather.
    """

    def __init__(self, eng, nsamples: int, nchans: int, *, group=None):
        import torch.distributed as dist

        from .engine import DeviceBuffer

        self.eng = eng
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nchans = nchans
        self.buf = DeviceBuffer(eng.device, (nsamples, nchans))
        handles = [None] * self.world
        dist.all_gather_object(handles, self.buf.ipc_handle(), group=group)
        self.peers: dict[int, int] = {}
        for r, h in enumerate(handles):
            if r != self.rank:
                p = ctypes.c_void_p()
                check(lib.pgb_ipc_open(eng.device, (ctypes.c_uint8 * 64).from_buffer_copy(h), ctypes.byref(p)))
                self.peers[r] = int(p.value)
        self.slices = row_slices(nsamples, self.world)

    @property
    def own_rows(self) -> tuple[int, int]:
        return self.slices[self.rank]

    def upload_own(self, host_rows: np.ndarray) -> int:
        """H2D of this rank's rows (host_rows = rows own_rows[0]:own_rows[1], ideally pinned)."""
        r0, r1 = self.own_rows
        nb = (r1 - r0) * self.nchans
        assert host_rows.nbytes == nb and host_rows.flags.c_contiguous
        self.eng.copy_async(self.buf.ptr + r0 * self.nchans, host_rows.ctypes.data, nb)
        return nb

    def exchange(self) -> int:
        """Wait until every rank's rows are resident, then pull the peers' rows (bytes pulled)."""
        import torch.distributed as dist

        self.eng.synchronize()
        dist.barrier(group=self.group)
        pulled = 0
        for r, ptr in self.peers.items():
            a, b = self.slices[r]
            nb = (b - a) * self.nchans
            self.eng.copy_async(self.buf.ptr + a * self.nchans, ptr + a * self.nchans, nb)
            pulled += nb
        return pulled

    def close(self) -> None:
        import torch.distributed as dist

        self.eng.synchronize()
        dist.barrier(group=self.group)  # no peer still reads our buffer
        for ptr in self.peers.values():
            check(lib.pgb_ipc_close(ctypes.c_void_p(ptr)))
        self.peers.clear()
        self.buf.free()


def search_file_distributed(payload, task, *, rank: int, world: int, device: int, group=None,
                            gather_device=None):
    """Sharded file search; rank 0 returns the SearchResult (candidates, clusters and the
    skipped pairs of every shard), other ranks None."""
    import torch

    from .engine import default_engine
    from .pipeline import SearchResult

    work = trial_work(task.plan, [c.length for c in task.chunks])
    lo, hi = shard_trials(work, world, DD_TRIAL_BLOCK)[rank]
    eng = default_engine(device)
    cands, _, skipped = eng.search_file(payload, task.header.nsamples, task.chunks, task.plan,
                                        task.engine, trial_range=(lo, hi), cluster=False, rfi=task.rfi)
    gdev = gather_device if gather_device is not None else torch.device("cuda", device)
    merged = gather_candidates(cands, device=gdev, group=group)
    all_skipped = gather_skipped(skipped, device=gdev, group=group)
    if rank != 0:
        return None
    clusters = eng.link_grid(merged, task.engine.radii)
    return SearchResult(merged, clusters, all_skipped)
