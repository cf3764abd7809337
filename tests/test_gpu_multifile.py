"""Multi-file execution (next row f3): concurrent device contexts give the same per-file
results as sequential searches, in submission order, with per-file error isolation."""
import numpy as np
import pytest

from paper_2512_00398_b200 import errors
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing
from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
from paper_2512_00398_b200.pipeline import SearchParams, create_task, run_multi_file, search_file, write_candidates

from .helpers import u8_chunk

pytestmark = pytest.mark.gpu


def _task(nch=128, n=1 << 15):
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=nch, tsamp=64e-6, nsamples=n)
    params = SearchParams(dm_lo=0.0, dm_hi=150.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=256), baseline_len_s=0.25, nsamps_chunk=1 << 14,
                          rfi=RfiConfig(False, False))
    return hdr, create_task(hdr, params)


def test_concurrent_files_match_sequential():
    hdr, task = _task()
    payloads = [u8_chunk(hdr, task.plan, hdr.nsamples, seed=2000 + i,
                         pulses=[(10 + 5 * i, 4000 + 1000 * i, 1 << (i % 5), 20.0)]) for i in range(8)]
    seq = [write_candidates(search_file(p, task).clusters) for p in payloads]
    par = run_multi_file(payloads, [task] * 8, n_exec=4)
    assert [write_candidates(r.clusters) for r in par] == seq
    assert all(s for s in seq)


def test_failing_file_is_isolated():
    hdr, task = _task()
    good = u8_chunk(hdr, task.plan, hdr.nsamples, seed=1)
    bad = np.zeros((10, hdr.nchans + 1), np.uint8)  # wrong channel count
    out = run_multi_file([good, bad, good], [task, task, task], n_exec=2)
    assert not isinstance(out[0], Exception) and not isinstance(out[2], Exception)
    assert isinstance(out[1], Exception)
    with pytest.raises(errors.ConfigError):
        run_multi_file([good], [task], n_exec=0)
