"""Bounded-memory streaming ingest (row f2): a search straight from an 8-bit SIGPROC file
on disk through pgb_stream_* (chunks read by parallel preads into two pinned buffers
while the previous chunk computes) produces exactly the reference's output.

* config A and config B files (tools/synth.py bytes) against the reference pipeline's
  golden results (tests/golden/config_<name>.npz, every candidate field, clusters,
  skipped pairs, .cand text);
* many small chunks, RFI on and off, against the whole-payload device search (itself
  pinned to the reference in test_gpu_configs.py / test_gpu_rfi.py);
* host memory stays at O(2 chunks): a subprocess searching the 4 GiB config-B file
  peaks well below the file size.
"""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from tests.helpers import FIELDS, task_for

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"

pytestmark = pytest.mark.gpu


def _params(cfg):
    from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
    from paper_2512_00398_b200.pipeline import LinearSpacing, SearchParams

    rfi = bool(cfg.get("rfi", False))
    return SearchParams(dm_lo=cfg["dm_lo"], dm_hi=cfg["dm_hi"], spacing=LinearSpacing(cfg["dm_step"]),
                        engine=EngineConfig(n_workers=1, detect_thresh=cfg["detect_thresh"],
                                            boxcar_max=cfg["boxcar_max"]),
                        baseline_len_s=cfg["baseline_s"], nsamps_chunk=cfg["nsamps_chunk"],
                        rfi=RfiConfig(narrowband=rfi, broadband=rfi))


def _assert_same(res, cands, clusters, skipped):
    for k in FIELDS:
        assert np.array_equal(res.candidates[k], cands[k]), k
    assert np.array_equal(res.clusters.records, clusters.records)
    assert np.array_equal(res.clusters.members, clusters.members)
    assert np.array_equal(np.asarray(res.skipped).reshape(-1, 2), np.asarray(skipped).reshape(-1, 2))


@pytest.mark.parametrize("name", ["A", pytest.param("B", marks=pytest.mark.slow)])
def test_search_fil_matches_reference_golden(tmp_path, name):
    from paper_2512_00398_b200.pipeline import search_fil, write_candidates
    from tools import synth

    gz = GOLDEN / f"config_{name}.npz"
    if not gz.exists():
        pytest.skip(f"{gz.name} not generated")
    z = np.load(gz)
    meta = json.loads(str(z["meta"]))
    cfg = meta["cfg"]
    task = task_for(cfg)
    path = tmp_path / f"{name}.fil"
    synth.write_filterbank(path, cfg, task.plan.delays)
    res = search_fil(path, _params(cfg))
    assert len(res.candidates) == meta["ncandidates"]
    if "candidates" in z.files:
        for k in FIELDS:
            assert np.array_equal(res.candidates[k], z["candidates"][k]), k
    zc, zm = z["clusters"], z["members"]
    for i in range(len(zc)):
        off, cnt = int(zc["member_offset"][i]), int(zc["members"][i])
        assert np.array_equal(res.clusters.member_ids(i), zm[off: off + cnt]), i
    assert write_candidates(res.clusters) == z["cand_text"].tobytes().decode()
    assert np.array_equal(np.asarray(res.skipped).reshape(-1, 2), z["skipped"].reshape(-1, 2))


@pytest.mark.parametrize("rfi", [False, True])
def test_search_fil_many_chunks_equals_payload_search(tmp_path, engine, rfi):
    """7 overlapping chunks (buffers alternate, uneven last chunk) with and without RFI."""
    from paper_2512_00398_b200.pipeline import search_fil
    from tools import synth

    cfg = dict(synth.CONFIGS["A"], nsamples=90000, nsamps_chunk=20000, boxcar_max=256, npulses=6,
               seed=77, rfi=rfi, dm_hi=200.0)
    task = task_for(cfg)
    assert len(task.chunks) >= 5
    path = tmp_path / "many.fil"
    synth.write_filterbank(path, cfg, task.plan.delays)
    res = search_fil(path, _params(cfg))
    payload = synth.payload(cfg, task.plan.delays)
    cands, clusters, skipped = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan,
                                                  task.engine, rfi=task.rfi)
    assert len(cands) > 0
    _assert_same(res, cands, clusters, skipped)


@pytest.mark.parametrize("read_threads", [1, 3, 16])
def test_first_chunk_pieces_any_count(tmp_path, engine, read_threads):
    """The first chunk is read and uploaded in max(2, read_threads) 64-row-aligned pieces and
    computed as they arrive: any piece count gives the whole-payload search's result."""
    from paper_2512_00398_b200.pipeline import search_fil
    from tools import synth

    cfg = dict(synth.CONFIGS["A"], nsamples=50000, nsamps_chunk=30000, boxcar_max=256, npulses=4,
               seed=78, dm_hi=150.0)
    task = task_for(cfg)
    path = tmp_path / "pieces.fil"
    synth.write_filterbank(path, cfg, task.plan.delays)
    res = search_fil(path, _params(cfg), read_threads=read_threads)
    payload = synth.payload(cfg, task.plan.delays)
    cands, clusters, skipped = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan,
                                                  task.engine)
    assert len(cands) > 0
    _assert_same(res, cands, clusters, skipped)


def test_unreadable_piece_fails_the_push(tmp_path, monkeypatch):
    """A piece of the first chunk that cannot be read is reported to the library
    (pgb_stream_upload_part with ok = 0): the push fails with pulsegrid::read_error instead of
    searching stale bytes, and the engine streams the next file normally."""
    import os

    from paper_2512_00398_b200.errors import ReadError
    from paper_2512_00398_b200.pipeline import search_fil
    from tools import synth

    cfg = dict(synth.CONFIGS["A"], nsamples=50000, nsamps_chunk=30000, boxcar_max=256, seed=79, dm_hi=150.0)
    task = task_for(cfg)
    path = tmp_path / "bad.fil"
    synth.write_filterbank(path, cfg, task.plan.delays)
    real = os.preadv
    bad_at = 15000 * cfg["nchans"]  # inside the first chunk

    def flaky(fd, bufs, off):
        if off <= bad_at < off + sum(len(b) for b in bufs):
            raise OSError("simulated read failure")
        return real(fd, bufs, off)

    monkeypatch.setattr(os, "preadv", flaky)
    with pytest.raises(ReadError):
        search_fil(path, _params(cfg), read_threads=4)
    monkeypatch.setattr(os, "preadv", real)
    res = search_fil(path, _params(cfg), read_threads=4)
    assert len(res.candidates) > 0


@pytest.mark.slow
def test_search_fil_host_memory_is_bounded(tmp_path):
    """Peak RSS of a process streaming the 4 GiB config-B file stays far below the file size
    (VmHWM of the fresh process: ru_maxrss would carry the forking parent's peak)."""
    from tools import synth

    cfg = dict(synth.CONFIGS["B"])
    task = task_for(cfg)
    path = tmp_path / "B.fil"
    synth.write_filterbank(path, cfg, task.plan.delays)
    code = f"""
import sys
sys.path.insert(0, {str(ROOT)!r})
from tests.test_gpu_stream import _params
from tools import synth
from paper_2512_00398_b200.pipeline import search_fil
res = search_fil({str(path)!r}, _params(dict(synth.CONFIGS['B'])))
hwm = [int(l.split()[1]) for l in open('/proc/self/status') if l.startswith('VmHWM:')][0]
print(len(res.candidates), hwm * 1024)
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    ncand, rss = map(int, out.stdout.split()[-2:])
    fsize = path.stat().st_size
    assert ncand > 0
    # two 1 GiB pinned chunk buffers + the CUDA/torch runtime; the file is 4 GiB
    assert rss < 0.8 * fsize, (rss, fsize)
