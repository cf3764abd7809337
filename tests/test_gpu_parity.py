"""GPU parity: the CUDA path (through the C ABI) against the CPU oracles.

Bar (BASELINE.json north_star): dedispersed sums bit-exact; candidate lists
identical in (dm_trial, peak_sample, width_index, begin, end) and -- because
every kernel reproduces the reference's rounding sequence -- snr bit-identical
too (the stated tolerance is 1e-4 relative; we assert equality and report the
tolerance form separately in test_snr_within_stated_tolerance).
"""
import numpy as np
import pytest

from paper_2512_00398_b200 import errors
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Chunk, ChunkSpec, EngineConfig, LinkRadii

from .helpers import assert_same_candidates, cfg_dict, clusters_equal, f32_chunk, random_candidates, u8_chunk

pytestmark = pytest.mark.gpu

DEDISP_CASES = [
    # nchans, fch1, foff, L, dm_hi, step
    (64, 1500.0, -2.0, 6000, 300.0, 5.0),
    (13, 1500.0, -7.0, 3000, 80.0, 3.0),
    (256, 1500.0, -1.0, 9000, 100.0, 1.0),
    (1024, 1500.0, -0.25, 20000, 500.0, 2.0),
    (4096, 1518.0, -0.0703125, 40000, 2000.0, 40.0),
    # wide per-block delay spreads: 4 and 2 channels per stage, 3-4 vectors per stager
    (4096, 1518.0, -0.0703125, 24000, 800.0, 8.0),
    (4096, 1518.0, -0.0703125, 30000, 1400.0, 14.0),
    # windows where three 8-channel ring slots do not fit but two do (2-slot ring)
    (4096, 1518.0, -0.0703125, 20000, 400.0, 4.0),
    (1, 1500.0, -1.0, 2000, 0.0, 1.0),
    (517, 1450.0, -0.5, 12000, 400.0, 2.5),
]


@pytest.mark.parametrize("nchans,fch1,foff,L,dm_hi,step", DEDISP_CASES)
def test_dedisperse_u8_bit_exact(engine, port, nchans, fch1, foff, L, dm_hi, step):
    hdr = FilterbankHeader(fch1=fch1, foff=foff, nchans=nchans, tsamp=64e-6)
    plan = generate_dm_trials(0.0, dm_hi, hdr, LinearSpacing(step))
    ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
    data = u8_chunk(hdr, plan, L, seed=nchans)
    got = engine.dedisperse(data, plan, range(0, len(ok)))
    f = data.astype(np.float32)
    for t in range(0, len(ok), max(1, len(ok) // 12)):
        want = port.dedisperse(f, plan.delays[t])
        assert np.array_equal(got[t], want), t


@pytest.mark.parametrize("nchans,L", [(16, 4096), (37, 5000), (300, 7000)])
def test_dedisperse_f32_bit_exact(engine, port, nchans, L):
    hdr = FilterbankHeader(fch1=1500.0, foff=-4.0 * 16 / nchans, nchans=nchans, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 200.0, hdr, LinearSpacing(11.0))
    data = f32_chunk(nchans, L, seed=nchans, scale=5.0)
    ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
    got = engine.dedisperse(data, plan, range(0, len(ok)))
    for t in ok:
        assert np.array_equal(got[t], port.dedisperse(data, plan.delays[t])), t


@pytest.mark.parametrize("nchans,foff,L,dm_hi,step", [
    (2048, -0.14, 24000, 800.0, 8.0),     # wide windows: fewer channels per ring stage
    (1000, -0.3, 20000, 1500.0, 33.0),    # 46 trials: a partial second block, nchans % 8 != 0
])
def test_dedisperse_f32_ring_wide_windows(engine, port, nchans, foff, L, dm_hi, step):
    """fp32 ring kernel (non-integer data): in-order fp32 sums bit-exact for sampled trials
    of plans whose per-block delay spreads force narrow stages."""
    hdr = FilterbankHeader(fch1=1500.0, foff=foff, nchans=nchans, tsamp=64e-6)
    plan = generate_dm_trials(0.0, dm_hi, hdr, LinearSpacing(step))
    data = f32_chunk(nchans, L, seed=nchans + 1, scale=5.0)
    ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
    got = engine.dedisperse(data, plan, range(0, len(ok)))
    for t in ok[::max(1, len(ok) // 8)] + [ok[-1]]:
        assert np.array_equal(got[t], port.dedisperse(data, plan.delays[t])), t


def test_dedisperse_chunk_too_short(engine):
    # tests/test_dedisp.cpp:245-257
    hdr = FilterbankHeader(fch1=1500.0, foff=-50.0, nchans=8, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 500.0, hdr, LinearSpacing(250.0))
    data = np.ones((64, 8), np.float32)
    with pytest.raises(errors.ChunkTooShortError) as ei:
        engine.dedisperse(data, plan, range(2, 3))
    assert ei.value.trial_index == 2


def _small_u8_case():
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=128, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 120.0, hdr, LinearSpacing(4.0))
    L = 12000
    data = u8_chunk(hdr, plan, L, seed=7, pulses=[(15, 3000, 8, 25.0), (22, 7000, 1, 14.0),
                                                   (5, 9500, 64, 18.0)])
    return hdr, plan, data


@pytest.mark.parametrize("window,bmax", [(2001, 256), (0, 64), (40001, 1024)])
def test_run_dm_loop_u8_vs_port(engine, port, window, bmax):
    hdr, plan, data = _small_u8_case()
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=bmax, baseline_window=window)
    spec = ChunkSpec.whole(data.shape[0])
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk = port.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


@pytest.mark.parametrize("bmax", [2048, 4096])
def test_run_dm_loop_runs_across_boxcar_tiles(engine, port, bmax):
    """Wide and narrow pulses straddling the boxcar tile boundaries (8192 outputs per
    tile at bmax 4096, 6144 at 2048): runs split into fragments must stitch back."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=128, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 60.0, hdr, LinearSpacing(4.0))
    L = 40000
    T = 8192 if bmax == 4096 else 6144
    data = u8_chunk(hdr, plan, L, seed=21, pulses=[(3, T - 40, 128, 30.0), (9, 2 * T - 3, 8, 25.0),
                                                   (12, 3 * T - 700, 1024, 40.0)])
    cfg = EngineConfig(n_workers=1, tsamp=hdr.tsamp, boxcar_max=bmax, baseline_window=8001)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk = port.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def test_run_dm_loop_u8_chunk_edges(engine, ref):
    """Interior chunk of a file: start > 0, overlap > 0, valid range < chunk
    (edge-run drops and valid-range filter, src/detect.cpp:235-238)."""
    hdr, plan, data = _small_u8_case()
    L = data.shape[0]
    spec = ChunkSpec(index=1, start_sample=50_000, length=L, overlap=2500, valid_begin=50_000,
                     valid_end=50_000 + L - 2500)
    cfg = EngineConfig(n_workers=4, tsamp=hdr.tsamp, boxcar_max=512, baseline_window=3001)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def test_run_dm_loop_config_a(engine, ref):
    """Config A of BASELINE.json: 1024 ch, 2^16 samples, DM 0-500 step 2 (251 trials),
    boxcar 4096, baseline 2 s, three injected pulses."""
    hdr = FilterbankHeader(fch1=1500.0, foff=-0.25, nchans=1024, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 500.0, hdr, LinearSpacing(2.0))
    L = 1 << 16
    data = u8_chunk(hdr, plan, L, seed=1000, pulses=[(50, 20000, 4, 12.0), (125, 40000, 16, 16.0),
                                                     (200, 52000, 64, 20.0)])
    cfg = EngineConfig(n_workers=16, tsamp=hdr.tsamp, boxcar_max=4096, baseline_window=31251)
    spec = ChunkSpec.whole(L)
    res = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 10
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def _float_workload(ref):
    """tests/test_engine.cpp:17-33: 32-ch float noise with two pulses."""
    fch1, foff, tsamp, nch, L = 1500.0, -2.0, 64e-6, 32, 8192
    g = ref.generate_noise(fch1, foff, tsamp, nch, L, 0.0, 1.0, 77)
    ref.inject_pulse(g, fch1, foff, tsamp, 100.0, 2000 * tsamp, 4, ref.amplitude_for_snr(18.0, 1.0, 32, 4))
    ref.inject_pulse(g, fch1, foff, tsamp, 40.0, 5000 * tsamp, 8, ref.amplitude_for_snr(15.0, 1.0, 32, 8))
    hdr = FilterbankHeader(fch1=fch1, foff=foff, nchans=nch, tsamp=tsamp)
    plan = generate_dm_trials(0.0, 150.0, hdr, LinearSpacing(2.0))
    return hdr, plan, g


def test_run_dm_loop_f32_engine_workload(engine, ref):
    hdr, plan, g = _float_workload(ref)
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=1001)
    spec = ChunkSpec.whole(g.shape[0])
    res = engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(g, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)
    best = res.candidates[np.argmax(res.candidates["snr"])]
    assert abs(best["dm"] - 100.0) <= 2.0 and abs(int(best["peak_sample"]) - 2000) <= 4


@pytest.mark.parametrize("window", [2001, 40001])
def test_f32_baseline_exact_and_replayed_rows(abl_engine, engine, ref, monkeypatch, window):
    """Float chunk of multiples of 1/8 (every trial's window sums exact in double -> the
    fixed-point baseline) with one fine-grained sample late in the zero-delay channel:
    trials short enough to exclude it stay exact, the rest take the sequential replay.
    Both mixes, and the all-sequential baseline, match the reference library."""
    hdr, plan, data = _small_u8_case()
    g = data.astype(np.float32) / np.float32(8.0)
    L = g.shape[0]
    zero_ch = int(np.argmin(plan.delays[-1]))
    g[L - 1 - 300, zero_ch] = np.float32(0.000123456)
    md = np.array([plan.trial_max_delay(t) for t in range(plan.ntrials)])
    assert (md > 300).any() and (md < 300).any()
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=256, baseline_window=window, detect_thresh=5.0)
    spec = ChunkSpec.whole(L)
    want, want_sk, _ = ref.run_dm_loop(g, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    a = engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    monkeypatch.setenv("PGB_BASELINE_SERIAL", "1")
    b = abl_engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    for r in (a, b):
        assert_same_candidates(r.candidates, want)
        assert np.array_equal(r.skipped_trials, want_sk)


def test_f32_baseline_subnormal_fixed_point(engine, ref):
    """Every value a multiple of 2^-140 below 2^-126 (subnormal floats): the trials pass the
    exactness check with L = -140 and run in fixed point; same candidates as the reference."""
    hdr, plan, data = _small_u8_case()
    g = (data.astype(np.float64) * 2.0 ** -140).astype(np.float32)
    assert np.all(np.abs(g) < np.float32(2.0 ** -126))
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=256, baseline_window=2001)
    spec = ChunkSpec.whole(g.shape[0])
    want, want_sk, _ = ref.run_dm_loop(g, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert len(want) > 0
    res = engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


def test_widened_u8_chunk_takes_integer_path(abl_engine, engine, port, monkeypatch):
    """A float chunk of 8-bit codes (read_chunk's widening) is repacked on the device;
    results equal the u8 path, the forced fp32 path and the oracle."""
    hdr, plan, data = _small_u8_case()
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=256, baseline_window=2001)
    spec = ChunkSpec.whole(data.shape[0])
    a = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    b = engine.run_dm_loop(Chunk(spec, data.astype(np.float32)), plan, cfg)
    monkeypatch.setenv("PGB_FORCE_F32_PATH", "1")
    c = abl_engine.run_dm_loop(Chunk(spec, data.astype(np.float32)), plan, cfg)
    want, _ = port.run_dm_loop(data, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    for r in (a, b, c):
        assert_same_candidates(r.candidates, want)


def test_snr_within_stated_tolerance(engine, ref):
    hdr, plan, g = _float_workload(ref)
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=1001)
    spec = ChunkSpec.whole(g.shape[0])
    res = engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    want, _, _ = ref.run_dm_loop(g, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    assert_same_candidates(res.candidates, want, exact_snr=False)


def test_degenerate_trials_are_skipped(engine):
    # tests/test_engine.cpp:158-170
    hdr = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=32, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 150.0, hdr, LinearSpacing(2.0))
    data = np.zeros((8192, 32), np.float32)
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=1001)
    res = engine.run_dm_loop(Chunk(ChunkSpec.whole(8192), data), plan, cfg)
    assert len(res.candidates) == 0
    assert np.array_equal(res.skipped_trials, np.arange(plan.ntrials))


def test_uncoverable_trials_are_skipped(engine, ref):
    # tests/test_engine.cpp:172-188
    hdr = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=32, tsamp=64e-6)
    g = ref.generate_noise(1500.0, -2.0, 64e-6, 32, 1024, 0.0, 1.0, 78)
    plan = generate_dm_trials(0.0, 2000.0, hdr, LinearSpacing(500.0))
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=101)
    res = engine.run_dm_loop(Chunk(ChunkSpec.whole(1024), g), plan, cfg)
    want, want_sk, _ = ref.run_dm_loop(g, vars(ChunkSpec.whole(1024)), plan.dms, plan.delays,
                                       cfg_dict(cfg))
    assert np.array_equal(res.skipped_trials, want_sk)
    assert_same_candidates(res.candidates, want)
    fits = [plan.trial_max_delay(t) < 1024 for t in range(plan.ntrials)]
    assert [t not in set(res.skipped_trials.tolist()) for t in range(plan.ntrials)] == fits


def test_timing_sink_skips_unprocessed_trials(engine, ref):
    """EngineConfig.timing_sink: one TrialTiming per trial that finished the chain, with the
    batched device stage times amortised over them (src/engine.cpp:147-213)."""
    from dataclasses import replace

    hdr = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=32, tsamp=64e-6)
    g = ref.generate_noise(1500.0, -2.0, 64e-6, 32, 1024, 0.0, 1.0, 78)
    plan = generate_dm_trials(0.0, 2000.0, hdr, LinearSpacing(500.0))
    recs = []
    cfg = replace(EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=101),
                  timing_sink=recs.append)
    res = engine.run_dm_loop(Chunk(ChunkSpec.whole(1024), g), plan, cfg)
    done = [t for t in range(plan.ntrials) if t not in set(res.skipped_trials.tolist())]
    assert 0 < len(done) < plan.ntrials
    assert [r.trial for r in recs] == done
    for r in recs:
        assert r.dedisperse_ms > 0 and r.baseline_ms > 0 and r.normalize_ms > 0 and r.boxcar_ms > 0
        assert r.peaks_ms >= 0


def test_config_errors(engine):
    hdr, plan, data = _small_u8_case()
    spec = ChunkSpec.whole(data.shape[0])
    with pytest.raises(errors.ConfigError):
        engine.run_dm_loop(Chunk(spec, data), plan, EngineConfig(n_workers=0, tsamp=hdr.tsamp))
    with pytest.raises(errors.ConfigError):
        engine.run_dm_loop(Chunk(spec, data), plan, EngineConfig(boxcar_max=48, tsamp=hdr.tsamp))
    with pytest.raises(errors.ConfigError):
        engine.run_dm_loop(Chunk(spec, data), plan,
                           EngineConfig(memory_budget=1000, tsamp=hdr.tsamp))


def test_link_grid_random_sets(engine, port):
    # tests/test_cluster.cpp:102-120 (200 random sets, random radii)
    rng = np.random.default_rng(31)
    for _ in range(60):
        n = int(rng.integers(1, 400))
        extent = int(rng.integers(1, 50000))
        cands = random_candidates(rng, n, extent)
        radii = LinkRadii(int(rng.integers(1, 6)), int(rng.integers(0, 12)), int(rng.integers(0, 4)))
        got = engine.link_grid(cands, radii)
        recs, members = port.link_grid(cands, (radii.sep_time, radii.sep_dm_trials, radii.sep_width))
        clusters_equal(got, recs, members)


def test_link_grid_vs_reference_library(engine, ref):
    rng = np.random.default_rng(47)
    cands = random_candidates(rng, 10000, 5_000_000)
    got = engine.link_grid(cands, LinkRadii())
    recs, members, _ = ref.link_grid(cands, (3, 9, 3))
    clusters_equal(got, recs, members)


@pytest.mark.parametrize("n,extent", [(3000, 20_000), (5120, 200_000), (12288, 2_000_000),
                                      (20000, 3_000_000)])
def test_link_grid_smem_and_global_forests_agree(abl_engine, engine, port, monkeypatch, n, extent):
    """link_grid's linking variants -- warp per candidate over a global forest (default),
    one CTA with everything staged in shared memory (<= 5120), one CTA with a shared-memory
    forest (<= 12288), thread per candidate over a global forest -- must all give the
    reference clusters (dense sets make big components and contended unions)."""
    rng = np.random.default_rng(n)
    cands = random_candidates(rng, n, extent)
    recs, members = port.link_grid(cands, (3, 9, 3))
    clusters_equal(engine.link_grid(cands, LinkRadii()), recs, members)  # warp per candidate
    for mode in ("PGB_LINK_SMEM2", "PGB_LINK_SMEM1", "PGB_LINK_GLOBAL"):
        monkeypatch.setenv(mode, "1")
        clusters_equal(abl_engine.link_grid(cands, LinkRadii()), recs, members)
        monkeypatch.delenv(mode)


def test_link_grid_ties(engine):
    # tests/test_cluster.cpp:92-100
    from paper_2512_00398_b200 import abi

    c = np.zeros(3, abi.CANDIDATE_DTYPE)
    for i, (snr, peak, trial) in enumerate([(10.0, 101, 4), (10.0, 100, 9), (10.0, 100, 2)]):
        c[i]["snr"], c[i]["peak_sample"], c[i]["dm_trial"] = snr, peak, trial
        c[i]["width_samples"] = 1
    cl = engine.link_grid(c, LinkRadii(30, 9, 3))
    assert len(cl) == 1
    assert cl.representatives["peak_sample"][0] == 100 and cl.representatives["dm_trial"][0] == 2


def test_link_grid_empty(engine):
    from paper_2512_00398_b200 import abi

    assert len(engine.link_grid(np.zeros(0, abi.CANDIDATE_DTYPE))) == 0
