"""Property tests mirroring the reference's own unit tests on this path.

* dedispersion: delta response (tests/test_dedisp.cpp:154-173), DM-0 = channel sums
  (:131-152), linearity (:226-243);
* engine: worker-count and in-flight invariance (tests/test_engine.cpp:70-84, :130-145);
* clustering: transitivity (tests/test_cluster.cpp:74-85) and partition invariance
  under permutation of the input (:141-163).
"""
import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Chunk, ChunkSpec, EngineConfig, LinkRadii

from .helpers import assert_same_candidates, random_candidates, u8_chunk

pytestmark = pytest.mark.gpu


def _plan(nch=96, dm_hi=200.0, step=5.0):
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.5, nchans=nch, tsamp=64e-6)
    return hdr, generate_dm_trials(0.0, dm_hi, hdr, LinearSpacing(step))


@pytest.mark.parametrize("u8", [True, False])
def test_delta_response(engine, u8):
    hdr, plan = _plan()
    L = 8000
    t0 = 1234
    trial = 17
    d = plan.delays[trial]
    grid = np.zeros((L, hdr.nchans), np.uint8 if u8 else np.float32)
    for c in range(hdr.nchans):
        grid[t0 + d[c], c] = 1  # one sample per channel on the trial's own sweep
    out = engine.dedisperse(grid, plan, range(trial, trial + 1))[0]
    want = np.zeros_like(out)
    want[t0] = hdr.nchans
    assert np.array_equal(out, want)


def test_dm0_trial_is_channel_sum(engine):
    hdr, plan = _plan()
    assert plan.dms[0] == 0.0 and not plan.delays[0].any()
    L = 5000
    g = u8_chunk(hdr, plan, L, seed=5)
    out = engine.dedisperse(g, plan, range(0, 1))[0]
    assert np.array_equal(out, g.astype(np.int64).sum(axis=1).astype(np.float32)[: len(out)])


def test_linearity(engine):
    """Small integer-valued float grids: every partial sum is exact, so D(a + b) = D(a) + D(b)
    bit for bit (the reference checks it with a tolerance)."""
    hdr, plan = _plan()
    L = 6000
    rng = np.random.default_rng(9)
    a = rng.integers(0, 100, (L, hdr.nchans)).astype(np.float32)
    b = rng.integers(-50, 50, (L, hdr.nchans)).astype(np.float32)
    trials = range(0, plan.ntrials)
    da, db, dab = (engine.dedisperse(x, plan, trials) for x in (a, b, a + b))
    for x, y, z in zip(da, db, dab):
        assert np.array_equal(z, x + y)


def test_worker_and_in_flight_invariance(engine):
    hdr, plan = _plan(nch=128, dm_hi=120.0, step=4.0)
    L = 12000
    data = u8_chunk(hdr, plan, L, seed=12, pulses=[(10, 3000, 8, 25.0), (25, 8000, 32, 20.0)])
    spec = ChunkSpec.whole(L)
    base = None
    for workers, in_flight in [(1, 0), (3, 0), (8, 8), (8, 1 << 20), (16, 0)]:
        cfg = EngineConfig(n_workers=workers, tsamp=hdr.tsamp, boxcar_max=512, baseline_window=2001,
                           max_in_flight=in_flight)
        res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
        if base is None:
            base = res
            assert len(res.candidates) > 0
        else:
            assert_same_candidates(res.candidates, base.candidates)
            assert np.array_equal(res.skipped_trials, base.skipped_trials)


def test_link_grid_transitivity(engine):
    from paper_2512_00398_b200 import abi

    # a ~ b and b ~ c with a !~ c (peaks 0, 3, 6 at width 1, sep_time 3): one cluster
    c = np.zeros(3, abi.CANDIDATE_DTYPE)
    for i, peak in enumerate([0, 3, 6]):
        c[i]["snr"], c[i]["peak_sample"], c[i]["dm_trial"], c[i]["width_samples"] = 8.0 + i, peak, 5, 1
    cl = engine.link_grid(c, LinkRadii(3, 9, 3))
    assert len(cl) == 1 and cl.records["members"][0] == 3


def test_link_grid_partition_is_permutation_invariant(engine):
    rng = np.random.default_rng(77)
    cands = random_candidates(rng, 3000, 40_000)
    perm = rng.permutation(len(cands))
    a = engine.link_grid(cands, LinkRadii())
    b = engine.link_grid(cands[perm], LinkRadii())
    assert len(a) == len(b)

    def partition(cl, ids):
        return sorted(tuple(sorted(int(ids[m]) for m in cl.member_ids(i))) for i in range(len(cl)))

    assert partition(a, np.arange(len(cands))) == partition(b, perm)


def test_more_than_65535_trials(engine, port):
    """Trial rows index CUDA grid x dimensions (not y, capped at 65535): a 70001-trial
    plan runs and matches the C restatement."""
    from .helpers import cfg_dict

    hdr = FilterbankHeader(fch1=1500.0, foff=-8.0, nchans=8, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 70.0, hdr, LinearSpacing(0.001))
    assert plan.ntrials > 65535
    L = 3000
    data = u8_chunk(hdr, plan, L, seed=4, pulses=[(30000, 1200, 4, 40.0)])
    cfg = EngineConfig(n_workers=1, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=501)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk = port.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)
