"""End-to-end parity at the BASELINE.json config shapes against the reference pipeline.

The golden files (tests/golden/config_<name>.npz, made by make_golden_configs.py from
the UNMODIFIED reference library in parity mode) hold the reference's full-file
output for the deterministic payloads of tools/synth.py.  Here the GPU box
regenerates the identical bytes (checked by sha256), runs the device file search
(`Engine.search_file`, the path `pgb_search_file_u8` exposes) and compares every
candidate field (snr included, exactly), the clusters with their member ids, the
skipped (chunk, trial) pairs and the .cand text byte for byte.

A  = full config-A file (1 chunk)           B  = full config-B file (5 chunks, 1001 trials)
C1 = 2^20 samples of the config-C band, 4001 trials (one chunk)
E1 = 2^19 samples of the config-E band, 4096 trials, dense RFI, RFI excision on
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from tests.helpers import FIELDS, task_for

GOLDEN = Path(__file__).resolve().parent / "golden"

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NAMES = [n for n in ("A", "B", "C1", "E1") if (GOLDEN / f"config_{n}.npz").exists()]


def _load(name):
    z = np.load(GOLDEN / f"config_{name}.npz")
    return json.loads(str(z["meta"])), z


def _compare_candidates(got, z, meta):
    assert len(got) == meta["ncandidates"], (len(got), meta["ncandidates"])
    if "candidates" in z.files:
        want = z["candidates"]
        for k in FIELDS:
            if not np.array_equal(got[k], want[k]):
                bad = np.nonzero(got[k] != want[k])[0][:5]
                raise AssertionError(f"field {k} differs at {bad}: got {got[k][bad]} want {want[k][bad]}")
    for k, d in meta["candidate_digests"].items():
        assert hashlib.sha256(np.ascontiguousarray(got[k]).tobytes()).hexdigest() == d, k


@pytest.mark.parametrize("name", NAMES)
def test_config_file_matches_reference(engine, name):
    from paper_2512_00398_b200.pipeline import write_candidates
    from tools import synth

    meta, z = _load(name)
    cfg = meta["cfg"]
    task = task_for(cfg)
    assert task.plan.ntrials == meta["ntrials"]
    payload = synth.payload(cfg, task.plan.delays)
    assert hashlib.sha256(payload.tobytes()).hexdigest() == meta["payload_sha256"], \
        "generator produced different bytes than the golden run"
    cands, clusters, skipped = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan,
                                                  task.engine, rfi=task.rfi)
    _compare_candidates(cands, z, meta)
    want_cl, want_mem = z["clusters"], z["members"]
    assert len(clusters.records) == len(want_cl)
    for k in FIELDS:
        assert np.array_equal(clusters.records["representative"][k], want_cl["representative"][k]), k
    for k in ("members", "begin_sample", "end_sample", "dm_lo", "dm_hi"):
        assert np.array_equal(clusters.records[k], want_cl[k]), k
    for i in range(len(want_cl)):  # member ids of each cluster
        off, cnt = int(want_cl["member_offset"][i]), int(want_cl["members"][i])
        assert np.array_equal(clusters.member_ids(i), want_mem[off: off + cnt]), i
    assert np.array_equal(np.asarray(skipped, np.uint64).reshape(-1, 2), z["skipped"].reshape(-1, 2))
    assert write_candidates(clusters) == z["cand_text"].tobytes().decode()
