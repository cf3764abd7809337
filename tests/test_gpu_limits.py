"""Inputs the reference accepts that round 1's device path rejected (missing #5).

* Wide trial blocks: with coarse DM steps a 32-trial block's channel delay spread no
  longer fits a staged shared-memory window (config-B band, DM 0-5000 step 60: spread
  27363 samples).  Such blocks run the direct dedispersion kernel; the last, narrower
  block of the same plan still runs the staged kernel.  u8 and fp32 chunks.
* boxcar_max above the shared-memory tile ladder (16384, 32768): the tile kernel stops
  at w = 4096 and boxcar_level_kernel doubles on in global memory.

Each is compared with the reference library (oracle/_ref, parity mode): candidate lists
field by field (snr exact), skipped trials, and dedispersed sums bit for bit.
"""
import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Chunk, ChunkSpec, EngineConfig

from .helpers import assert_same_candidates, cfg_dict

pytestmark = pytest.mark.gpu


def _payload(hdr, plan, L, seed, pulses):
    from tools import synth

    cfg = dict(nchans=hdr.nchans, seed=seed, nsamples=L, npulses=0)
    data = synth.noise(hdr.nchans, seed, 0, L)
    for trial, t0, width, snr in pulses:
        amp = snr * 16.0 / np.sqrt(hdr.nchans * width)
        d = plan.delays[trial].astype(np.int64)
        cols = np.arange(hdr.nchans)
        for w in range(width):
            r = t0 + d + w
            keep = r < L
            v = data[r[keep], cols[keep]].astype(np.float64) + amp
            data[r[keep], cols[keep]] = np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8)
    del cfg
    return data


def _wide_case():
    hdr = FilterbankHeader(fch1=1518.0, foff=-0.0703125, nchans=4096, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 5000.0, hdr, LinearSpacing(60.0))
    return hdr, plan


def test_wide_blocks_exist_in_the_case():
    """The plan really has blocks beyond the staging capacity (and one that fits)."""
    from paper_2512_00398_b200._native import lib  # noqa: F401  (library present)

    hdr, plan = _wide_case()
    spreads = []
    for b in range(0, plan.ntrials, 32):
        d = plan.delays[b: b + 32]
        spreads.append(int((d.max(axis=0) - d.min(axis=0)).max()))
    assert max(spreads) == 27363 and min(spreads) < 20000, spreads


def test_wide_blocks_u8_run_dm_loop_matches_reference(engine, ref):
    hdr, plan = _wide_case()
    L = 1 << 17
    data = _payload(hdr, plan, L, 606, [(10, 20000, 8, 30.0), (40, 40000, 2, 25.0), (70, 3000, 64, 40.0)])
    cfg = EngineConfig(n_workers=16, tsamp=hdr.tsamp, boxcar_max=1024, baseline_window=31251)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def test_wide_blocks_dedispersed_sums_bit_exact(engine, port):
    hdr, plan = _wide_case()
    L = 1 << 17
    data = _payload(hdr, plan, L, 607, [])
    ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
    got = engine.dedisperse(data, plan, range(0, len(ok)))
    f = data.astype(np.float32)
    for t in [0, 5, 31, 32, 47, 63, 64, len(ok) - 1]:
        assert np.array_equal(got[t], port.dedisperse(f, plan.delays[t])), t


def test_wide_blocks_f32_match_reference(engine, ref, port):
    """Non-integer chunk (fp32 in-order path) with wide blocks: 256 channels over 512 MHz,
    DM step 25 -> 32-trial spreads of ~29k samples."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=256, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 2000.0, hdr, LinearSpacing(25.0))
    L = 1 << 17
    rng = np.random.default_rng(5)
    data = (rng.standard_normal((L, hdr.nchans)) * 3.0).astype(np.float32)
    d = plan.delays[20]
    for c in range(hdr.nchans):
        data[30000 + d[c]: 30000 + d[c] + 16, c] += 2.5
    ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
    got = engine.dedisperse(data, plan, range(0, len(ok)))
    for t in [0, 20, 31, 32, 63, len(ok) - 1]:
        assert np.array_equal(got[t], port.dedisperse(data, plan.delays[t])), t
    cfg = EngineConfig(n_workers=16, tsamp=hdr.tsamp, boxcar_max=512, baseline_window=4001)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


@pytest.mark.parametrize("bmax", [16384, 32768])
def test_boxcar_max_above_tile_ladder(engine, ref, bmax):
    """Very wide pulses found at widths 8192-32768 (levels 13-15 in global memory), runs
    crossing the level kernel's strips, pulses near the chunk ends."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-0.25, nchans=1024, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 120.0, hdr, LinearSpacing(4.0))
    L = 1 << 17
    data = _payload(hdr, plan, L, 808, [(5, 10000, 8192, 60.0), (20, 60000, 16384, 90.0),
                                        (25, 100000, 4096, 40.0), (12, 200, 32, 20.0)])
    cfg = EngineConfig(n_workers=16, tsamp=hdr.tsamp, boxcar_max=bmax, baseline_window=0)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert (want["width_index"] >= 13).any()  # the global levels produced candidates
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def test_boxcar_max_above_tile_ladder_interior_chunk(engine, ref):
    """Interior chunk (edge-run drops, valid range) with boxcar_max 16384."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-0.25, nchans=1024, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 120.0, hdr, LinearSpacing(4.0))
    L = 1 << 17
    # (amplitudes above half a code: smaller ones vanish in the round-half-up quantisation)
    data = _payload(hdr, plan, L, 809, [(7, 1000, 16384, 500.0), (9, 70000, 8192, 350.0),
                                        (3, L - 20000, 16384, 500.0)])
    spec = ChunkSpec(index=2, start_sample=300000, length=L, overlap=20000, valid_begin=300000,
                     valid_end=300000 + L - 20000)
    cfg = EngineConfig(n_workers=16, tsamp=hdr.tsamp, boxcar_max=16384, baseline_window=65537)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert (want["width_index"] >= 13).any()
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)
