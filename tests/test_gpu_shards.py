"""DM-trial sharding (multi-GPU path) on one device: the per-shard candidate lists,
merged and re-sorted the way distributed.gather_candidates does on rank 0, equal the
single-device list, and link_grid of the merge equals link_grid of the whole."""
import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing
from paper_2512_00398_b200.distributed import shard_trials, sort_candidates, trial_work
from paper_2512_00398_b200.engine import Engine, EngineConfig, RfiConfig
from paper_2512_00398_b200.pipeline import SearchParams, create_task

from .helpers import FIELDS, u8_chunk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_search_equals_single_device(world):
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=256, tsamp=64e-6, nsamples=1 << 16)
    params = SearchParams(dm_lo=0.0, dm_hi=300.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=1024), baseline_len_s=0.5,
                          nsamps_chunk=1 << 14, rfi=RfiConfig(False, False))
    task = create_task(hdr, params)
    payload = u8_chunk(hdr, task.plan, hdr.nsamples, seed=5,
                       pulses=[(30, 9000, 4, 22.0), (90, 30000, 32, 18.0), (140, 50000, 1, 16.0)])
    with Engine(0) as eng:
        full_c, full_cl, full_sk = eng.search_file(payload, hdr.nsamples, task.chunks, task.plan, task.engine)
        parts = []
        for lo, hi in shard_trials(trial_work(task.plan, [c.length for c in task.chunks]), world):
            c, _, _ = eng.search_file(payload, hdr.nsamples, task.chunks, task.plan, task.engine,
                                      trial_range=(lo, hi), cluster=False)
            parts.append(c)
        merged = sort_candidates(np.concatenate(parts).astype(full_c.dtype))
        assert len(full_c) > 0 and len(merged) == len(full_c)
        for k in FIELDS:
            assert np.array_equal(merged[k], full_c[k]), k
        cl = eng.link_grid(merged, task.engine.radii)
        assert np.array_equal(cl.records["members"], full_cl.records["members"])
        assert np.array_equal(cl.representatives["peak_sample"], full_cl.representatives["peak_sample"])
