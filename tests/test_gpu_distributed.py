"""The multi-GPU path end to end on one GPU: two ranks (processes) share cuda:0 over gloo.

Each rank uploads half of the file's rows into its own device buffer and pulls the other
half from its peer through CUDA IPC (PayloadFanout), searches its DM-trial shard, and
rank 0 gathers candidates and skipped (chunk, trial) pairs and clusters them
(search_file_distributed).  The result must equal the single-device search exactly,
with RFI excision on (the shard search once dropped the RFI settings) and
with skipped trials spread over both shards.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.helpers import FIELDS, task_for

pytestmark = pytest.mark.gpu

CASES = {
    # 5 overlapping chunks, RFI excision on (bursts + hot channels)
    "rfi_multichunk": dict(nsamples=90000, nsamps_chunk=30000, dm_hi=300.0, rfi=True),
    # one short chunk: trials whose delay span exceeds it are skipped (both shards hold some)
    "skipped_trials": dict(nsamples=5000, nsamps_chunk=1 << 18, dm_hi=500.0, rfi=False),
}


def _cfg(name):
    from tools import synth

    return dict(synth.CONFIGS["A"], boxcar_max=256, npulses=6, seed=91, **CASES[name])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2512_00398_b200.distributed import PayloadFanout, search_file_distributed
    from paper_2512_00398_b200.engine import default_engine
    from tests.helpers import task_for as tf
    from tools import synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg(name)
        task = tf(cfg)
        eng = default_engine(0)
        fan = PayloadFanout(eng, cfg["nsamples"], cfg["nchans"])
        r0, r1 = fan.own_rows
        host = np.ascontiguousarray(synth.payload(cfg, task.plan.delays, r0, r1 - r0))
        fan.upload_own(host)
        fan.exchange()
        eng.synchronize()
        res = search_file_distributed(fan.buf, task, rank=rank, world=world, device=0,
                                      gather_device=torch.device("cpu"))
        fan.close()
        if rank == 0:
            out_q.put((res.candidates.tobytes(), res.clusters.records.tobytes(), res.clusters.members.tobytes(),
                       np.asarray(res.skipped, np.uint64).tobytes()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", sorted(CASES))
def test_two_ranks_on_one_gpu_equal_single_device(engine, name):
    from paper_2512_00398_b200 import abi
    from tools import synth

    cfg = _cfg(name)
    task = task_for(cfg)
    payload = synth.payload(cfg, task.plan.delays)
    cands, clusters, skipped = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan,
                                                  task.engine, rfi=task.rfi)
    assert len(cands) > 0
    if name == "skipped_trials":
        assert len(skipped) > 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    c_b, cl_b, m_b, s_b = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = np.frombuffer(c_b, abi.CANDIDATE_DTYPE)
    assert len(got) == len(cands)
    for k in FIELDS:
        assert np.array_equal(got[k], cands[k]), k
    assert np.array_equal(np.frombuffer(cl_b, abi.CLUSTER_DTYPE), clusters.records)
    assert np.array_equal(np.frombuffer(m_b, np.uint64), clusters.members)
    assert np.array_equal(np.frombuffer(s_b, np.uint64).reshape(-1, 2), np.asarray(skipped).reshape(-1, 2))
