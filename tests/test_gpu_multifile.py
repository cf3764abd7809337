"""Multi-file execution (row f3, src/pipeline.cpp:121-219).

* run_multi_file on a batch of 10 8-bit files on disk (two creation workers, four
  execution workers over bounded queues, each executor a device context streaming its
  files with bounded memory): every .cand file is byte-identical to the reference's own
  create_task + execute_task on the same file (oracle/_ref, parity mode), FileOutcome
  carries status, cluster count, skipped pairs and stage times, in submission order;
* a missing file and a malformed file are isolated into their outcomes while the rest
  of the batch completes; zero workers raise config_error;
* the in-memory variant (search_payloads) equals sequential searches.
"""
import numpy as np
import pytest

from paper_2512_00398_b200 import errors
from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
from paper_2512_00398_b200.pipeline import (LinearSpacing, SearchParams, assign_output_paths, create_task,
                                            run_multi_file, search_file, search_payloads, write_candidates,
                                            write_summary)

from .helpers import task_for

pytestmark = pytest.mark.gpu

NFILES = 10


def _cfg(i):
    from tools import synth

    return dict(synth.CONFIGS["A"], nchans=256, nsamples=40000 + 3000 * i, nsamps_chunk=1 << 14,
                dm_hi=150.0, boxcar_max=256, npulses=3, seed=2000 + i, rfi=(i % 3 == 0))


def _params(cfg):
    rfi = bool(cfg.get("rfi"))
    return SearchParams(dm_lo=cfg["dm_lo"], dm_hi=cfg["dm_hi"], spacing=LinearSpacing(cfg["dm_step"]),
                        engine=EngineConfig(n_workers=4, detect_thresh=cfg["detect_thresh"],
                                            boxcar_max=cfg["boxcar_max"]),
                        baseline_len_s=0.25, nsamps_chunk=cfg["nsamps_chunk"],
                        rfi=RfiConfig(narrowband=rfi, broadband=rfi))


@pytest.fixture(scope="module")
def batch(tmp_path_factory):
    from tools import synth

    d = tmp_path_factory.mktemp("batch")
    paths = []
    for i in range(NFILES):
        cfg = _cfg(i)
        p = d / f"beam{i:02d}.fil"
        synth.write_filterbank(p, cfg, task_for(cfg).plan.delays)
        paths.append(str(p))
    return d, paths


def test_batch_cand_files_match_reference_execute_task(batch, ref, tmp_path):
    d, paths = batch
    # one shared SearchParams per batch, like the reference; RFI on for the whole batch
    # here, so files 0, 3, 6, 9 (dense synthetic RFI) and the clean ones both go through it
    cfg0 = dict(_cfg(0), rfi=True)
    params = _params(cfg0)
    out_dir = tmp_path / "cands"
    summary = run_multi_file(paths, params, str(out_dir), n_create=2, n_exec=4)
    assert summary.n_failed == 0, write_summary(summary)
    assert [f.path for f in summary.files] == paths
    for i, (p, f) in enumerate(zip(paths, summary.files)):
        assert f.ok and f.output_path == assign_output_paths(paths, str(out_dir))[i]
        want_path = tmp_path / f"ref{i}.cand"
        ncl, _ = ref.execute_file(p, want_path, dm_lo=cfg0["dm_lo"], dm_hi=cfg0["dm_hi"], dm_step=cfg0["dm_step"],
                                  n_workers=4, detect_thresh=cfg0["detect_thresh"], boxcar_max=cfg0["boxcar_max"],
                                  baseline_len_s=0.25, nsamps_chunk=cfg0["nsamps_chunk"], rfi_narrowband=True,
                                  rfi_broadband=True, parity=True)
        got = open(f.output_path, "rb").read()
        assert got == want_path.read_bytes(), p
        assert f.candidates == ncl > 0
        assert f.wall_ms > 0 and f.dm_loop_ms > 0 and f.cluster_ms >= 0 and f.write_ms >= 0
    assert summary.total_wall_ms > 0
    assert write_summary(summary).count("\tok\t") == NFILES


def test_failing_files_are_isolated(batch, tmp_path):
    d, paths = batch
    bad = d / "malformed.fil"
    bad.write_bytes(b"not a filterbank")
    batch_paths = [paths[0], str(d / "missing.fil"), str(bad), paths[1]]
    s = run_multi_file(batch_paths, _params(_cfg(1)), str(tmp_path / "o"), n_create=1, n_exec=2)
    assert [f.ok for f in s.files] == [True, False, False, True]
    assert s.n_failed == 2 and all(f.error for f in s.files if not f.ok)
    with pytest.raises(errors.ConfigError):
        run_multi_file(paths[:1], _params(_cfg(1)), str(tmp_path / "o2"), n_create=1, n_exec=0)


def test_assign_output_paths_numbers_repeated_stems():
    assert assign_output_paths(["/a/x.fil", "/b/x.fil", "/c/y.fil", "/d/x.fil"], "/o") == [
        "/o/x.cand", "/o/x.2.cand", "/o/y.cand", "/o/x.3.cand"]


def test_search_payloads_match_sequential():
    from paper_2512_00398_b200.dedisp import FilterbankHeader
    from tools import synth

    cfg = _cfg(1)
    hdr = FilterbankHeader(fch1=cfg["fch1"], foff=cfg["foff"], nchans=cfg["nchans"], tsamp=cfg["tsamp"],
                           nsamples=cfg["nsamples"])
    task = create_task(hdr, _params(cfg))
    payloads = [synth.payload(dict(cfg, seed=3000 + i, npulses=2), task.plan.delays) for i in range(8)]
    seq = [write_candidates(search_file(p, task).clusters) for p in payloads]
    par = search_payloads(payloads, [task] * 8, n_exec=4, devices=(0, 0))
    assert [write_candidates(r.clusters) for r in par] == seq
    bad = search_payloads([payloads[0], np.zeros((10, cfg["nchans"] + 1), np.uint8)], [task, task], n_exec=2)
    assert not isinstance(bad[0], Exception) and isinstance(bad[1], Exception)
