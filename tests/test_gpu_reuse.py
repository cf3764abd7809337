"""Overlap reuse in the file search: the outputs chunk k-1 already dedispersed for the
samples chunk k shares with it are moved, not summed again.  With and without the reuse
(PGB_NO_OVERLAP_REUSE=1 in the ablation library) the file's candidates and clusters must be identical, with the
baseline on (chain reads the slot's baseline buffer) and off (chain reads the series)."""
import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing
from paper_2512_00398_b200.engine import Engine, EngineConfig, RfiConfig, default_engine
from paper_2512_00398_b200.pipeline import SearchParams, SearchResult, create_task, search_file, write_candidates

from .helpers import u8_chunk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("baseline_s", [0.25, 0.0])
def test_reuse_matches_full_recompute(monkeypatch, baseline_s):
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=256, tsamp=64e-6, nsamples=1 << 16)
    params = SearchParams(dm_lo=0.0, dm_hi=300.0, spacing=LinearSpacing(2.0),
                          # without a baseline the normalised series sits near 1, so v ~ sqrt(w):
                          # threshold 4 makes the width-16 runs a dense, noise-driven set
                          engine=EngineConfig(boxcar_max=1024, detect_thresh=6.0 if baseline_s else 4.0),
                          baseline_len_s=baseline_s,
                          nsamps_chunk=1 << 14, rfi=RfiConfig(False, False))
    task = create_task(hdr, params)
    assert len(task.chunks) > 3
    payload = u8_chunk(hdr, task.plan, hdr.nsamples, seed=77,
                       pulses=[(40, 11000, 8, 25.0), (90, 23500, 32, 18.0), (140, 47000, 2, 30.0)])
    a = search_file(payload, task)
    adds_a = default_engine(0).last_dedisp_time()[2]
    monkeypatch.setenv("PGB_NO_OVERLAP_REUSE", "1")
    with Engine(0, ablations=True) as abl:
        cb, clb, _ = abl.search_file(payload, hdr.nsamples, task.chunks, task.plan, task.engine)
        adds_b = abl.last_dedisp_time()[2]
    b = SearchResult(cb, clb, None)
    assert adds_a < 0.95 * adds_b  # the reuse actually happened
    assert len(a.candidates) == len(b.candidates) > 0
    for k in a.candidates.dtype.names:
        assert np.array_equal(a.candidates[k], b.candidates[k]), k
    assert write_candidates(a.clusters) == write_candidates(b.clusters)


def test_progressive_first_chunk_matches(monkeypatch):
    """A host payload's first chunk is uploaded in pieces and its transpose and
    dedispersion start on the tiles whose samples arrived; the result must equal the
    one-piece upload (PGB_NO_PROGRESSIVE=1) and the device-resident payload."""
    import torch

    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=256, tsamp=64e-6, nsamples=3 << 15)
    params = SearchParams(dm_lo=0.0, dm_hi=300.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=1024), baseline_len_s=0.25,
                          nsamps_chunk=1 << 16, rfi=RfiConfig(False, False))
    task = create_task(hdr, params)
    payload = u8_chunk(hdr, task.plan, hdr.nsamples, seed=78,
                       pulses=[(30, 9000, 4, 25.0), (100, 40000, 16, 20.0), (140, 70000, 64, 30.0)])
    a = search_file(payload, task)
    monkeypatch.setenv("PGB_NO_PROGRESSIVE", "1")
    with Engine(0, ablations=True) as abl:
        cb, clb, _ = abl.search_file(payload, hdr.nsamples, task.chunks, task.plan, task.engine)
    b = SearchResult(cb, clb, None)
    monkeypatch.delenv("PGB_NO_PROGRESSIVE")
    c = search_file(torch.from_numpy(payload).cuda(), task)
    assert len(a.candidates) > 0
    for other in (b, c):
        assert len(other.candidates) == len(a.candidates)
        for k in a.candidates.dtype.names:
            assert np.array_equal(a.candidates[k], other.candidates[k]), k
        assert write_candidates(other.clusters) == write_candidates(a.clusters)


@pytest.mark.parametrize("alt", ["PGB_SYNC_BACK", "PGB_BACK_MAIN"])
@pytest.mark.parametrize("initial_cap", [None, "64"])
def test_async_back_halves_match_sync(monkeypatch, initial_cap, alt):
    """The file search's back halves run without host round trips (device-side counts,
    one read per file) on their own stream beside the next chunk's dedispersion; the result
    must equal the per-chunk synchronous path (PGB_SYNC_BACK=1) and the back halves on the
    main stream (PGB_BACK_MAIN=1), also when tiny initial buffers force the
    overflow-and-retry path."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=256, tsamp=64e-6, nsamples=3 << 15)
    params = SearchParams(dm_lo=0.0, dm_hi=300.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=1024), baseline_len_s=0.25,
                          nsamps_chunk=1 << 15, rfi=RfiConfig(False, False))
    task = create_task(hdr, params)
    payload = u8_chunk(hdr, task.plan, hdr.nsamples, seed=79,
                       pulses=[(30, 9000, 4, 25.0), (100, 40000, 512, 40.0), (140, 70000, 64, 30.0)])
    if initial_cap:
        monkeypatch.setenv("PGB_INITIAL_CAP", initial_cap)
    res = []
    for sync in (False, True):
        if sync:
            monkeypatch.setenv(alt, "1")
        with Engine(0, ablations=sync) as eng:  # both are ablation switches
            res.append(eng.search_file(payload, hdr.nsamples, task.chunks, task.plan, task.engine))
    (a, ca, sa), (b, cb, sb) = res
    assert len(a) == len(b) > 0
    for k in a.dtype.names:
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(ca.records, cb.records) and np.array_equal(sa, sb)
