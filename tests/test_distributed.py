"""The multi-GPU host logic on CPU: trial shards and the candidate gather (gloo, world 2).

On the B200 box the same code runs one rank per GPU with NCCL; here the device
search of each shard is replaced by the oracle (same candidates by construction),
and we check that gathering the shards' sorted lists and re-sorting reproduces the
single-device list exactly, so link_grid sees identical input for any world size.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_00398_b200 import abi
from paper_2512_00398_b200.distributed import shard_trials, sort_candidates, trial_work

from .helpers import random_candidates


def test_shard_trials_balance():
    rng = np.random.default_rng(0)
    w = rng.uniform(1, 10, 1001)
    for world in (1, 2, 3, 4, 8):
        shards = shard_trials(w, world)
        assert shards[0][0] == 0 and shards[-1][1] == 1001
        assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
        assert all(hi > lo for lo, hi in shards)
        loads = [w[lo:hi].sum() for lo, hi in shards]
        assert max(loads) - min(loads) <= 2 * w.max()


def test_trial_work_counts_coverable_samples():
    from paper_2512_00398_b200.dedisp import DmTrialPlan

    plan = DmTrialPlan(np.array([0.0, 1.0, 2.0]), np.array([[0, 5], [0, 50], [0, 500]]))
    w = trial_work(plan, [100, 40])
    assert list(w) == [2 * (95 + 35), 2 * (50 + 0), 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, full_bytes, out_q):
    import torch.distributed as dist

    from paper_2512_00398_b200.distributed import gather_candidates

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = np.frombuffer(full_bytes, abi.CANDIDATE_DTYPE)
    work = np.ones(200)
    lo, hi = shard_trials(work, world)[rank]
    mine = sort_candidates(full[(full["dm_trial"] >= lo) & (full["dm_trial"] < hi)])
    merged = gather_candidates(mine)
    if rank == 0:
        out_q.put(merged.tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_reproduces_single_device_order(world):
    rng = np.random.default_rng(4)
    full = random_candidates(rng, 500, 30000, ntrials=200)
    # make the (peak, trial, width) keys unique like run_dm_loop's
    full = full[np.unique(np.stack([full["peak_sample"], full["dm_trial"], full["width_index"]]),
                          axis=1, return_index=True)[1]]
    want = sort_candidates(full)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, full.tobytes(), q)) for r in range(world)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=120), abi.CANDIDATE_DTYPE)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got) == len(want)
    for k in abi.CANDIDATE_DTYPE.names:  # field by field (padding bytes are unspecified)
        assert np.array_equal(got[k], want[k]), k


def test_shard_trials_block_granule():
    """Shards on 32-trial dedispersion blocks: every boundary a multiple of 32, all trials
    covered once, block-cost balance within one block."""
    rng = np.random.default_rng(1)
    w = np.sort(rng.uniform(5, 10, 1001))[::-1].copy()  # work falls with DM
    for world in (2, 4, 8):
        shards = shard_trials(w, world, 32)
        assert shards[0][0] == 0 and shards[-1][1] == 1001
        assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
        assert all(lo % 32 == 0 and hi > lo for lo, hi in shards)
        cost = [32 * sum(w[b:b + 32].max() for b in range(lo, hi, 32)) for lo, hi in shards]
        assert max(cost) - min(cost) <= 2 * 32 * w.max()
    assert shard_trials(w[:40], 4, 32) == shard_trials(w[:40], 4)  # too few blocks: plain split


def _skip_worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_2512_00398_b200.distributed import gather_skipped

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # shard r skipped trials r, r+2, ... of chunks 0 and 3 (listed chunk-major per shard)
    mine = np.array([(c, t) for c in (0, 3) for t in range(rank, 12, world)], np.uint64)
    merged = gather_skipped(mine if rank else mine[:0].reshape(0, 2))  # rank 0 skipped none
    if rank == 0:
        out_q.put(merged.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_skipped_pairs_sorted_by_chunk_then_trial():
    """the (chunk, trial) skipped pairs of every shard reach rank 0, ordered like
    FileOutcome::skipped_trials (chunk by chunk, trials ascending)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_skip_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=120), np.uint64).reshape(-1, 2)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.array(sorted((c, t) for c in (0, 3) for t in range(12) if t % world != 0), np.uint64)
    assert np.array_equal(got, want)
