"""Synthetic inputs for the parity tests (numpy, seeded)."""
from __future__ import annotations

import numpy as np

from paper_2512_00398_b200 import abi
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials


def u8_chunk(hdr: FilterbankHeader, plan, L: int, seed: int, pulses=(), mean=100.0, sigma=16.0):
    """N(mean, sigma) noise quantised round-half-up to u8, plus dispersed top-hats.

    pulses: iterable of (trial_index, t0_sample, width, snr); the track follows the
    plan's own delays for that trial (matched trial)."""
    rng = np.random.default_rng(seed)
    grid = rng.normal(mean, sigma, (L, hdr.nchans))
    for trial, t0, width, snr in pulses:
        amp = snr * sigma / np.sqrt(hdr.nchans * width)
        d = plan.delays[trial]
        for c in range(hdr.nchans):
            s = t0 + int(d[c])
            grid[s: s + width, c] += amp
    return np.clip(np.floor(grid + 0.5), 0, 255).astype(np.uint8)


def f32_chunk(nchans: int, L: int, seed: int, scale: float = 1.0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((L, nchans)) * scale).astype(np.float32)


def cfg_dict(cfg) -> dict:
    return dict(n_workers=cfg.n_workers, tsamp=cfg.tsamp, detect_thresh=cfg.detect_thresh,
                boxcar_max=cfg.boxcar_max, baseline_window=cfg.baseline_window,
                memory_budget=cfg.memory_budget, max_in_flight=cfg.max_in_flight)


FIELDS = ("peak_sample", "dm_trial", "width_index", "begin_sample", "end_sample", "width_samples",
          "snr", "time_s", "dm")


def assert_same_candidates(got: np.ndarray, want: np.ndarray, *, exact_snr: bool = True):
    assert got.dtype == abi.CANDIDATE_DTYPE and want.dtype == abi.CANDIDATE_DTYPE
    assert len(got) == len(want), f"{len(got)} candidates vs {len(want)} expected"
    for k in FIELDS:
        if k == "snr" and not exact_snr:
            np.testing.assert_allclose(got[k], want[k], rtol=1e-4)
            continue
        if not np.array_equal(got[k], want[k]):
            bad = np.nonzero(got[k] != want[k])[0][:5]
            raise AssertionError(f"field {k} differs at {bad}: got {got[k][bad]} want {want[k][bad]}")


def random_candidates(rng, n: int, extent: int, ntrials: int = 200, nwidths: int = 8):
    """tests/test_cluster.cpp:28-36 shape: snr U(6,40), random peak/trial/width."""
    c = np.zeros(n, abi.CANDIDATE_DTYPE)
    c["snr"] = rng.uniform(6.0, 40.0, n).astype(np.float32)
    c["peak_sample"] = rng.integers(0, extent, n)
    c["dm_trial"] = rng.integers(0, ntrials, n)
    c["width_index"] = rng.integers(0, nwidths, n)
    c["width_samples"] = np.left_shift(1, c["width_index"].astype(np.uint64))
    c["dm"] = 0.5 * c["dm_trial"]
    c["begin_sample"] = np.where(c["peak_sample"] > 2, c["peak_sample"] - 2, 0)
    c["end_sample"] = c["peak_sample"] + 2
    c["time_s"] = c["peak_sample"] * 64e-6
    return c


def clusters_equal(got, want_recs: np.ndarray, want_members: np.ndarray):
    """Compare product Clusters with an oracle (records, flat members) pair."""
    assert len(got.records) == len(want_recs), (len(got.records), len(want_recs))
    gr, wr = got.records, want_recs
    for k in FIELDS:
        assert np.array_equal(gr["representative"][k], wr["representative"][k]), k
    for k in ("members", "begin_sample", "end_sample", "dm_lo", "dm_hi"):
        assert np.array_equal(gr[k], wr[k]), k
    for i in range(len(wr)):
        a = got.member_ids(i)
        off, cnt = int(wr["member_offset"][i]), int(wr["members"][i])
        assert np.array_equal(a, want_members[off: off + cnt]), i


def task_for(cfg: dict):
    """The product's create_task for a tools/synth.py config dict (reference defaults
    otherwise: one worker, link radii 3/9/3; RFI on exactly when the config says so)."""
    from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
    from paper_2512_00398_b200.pipeline import SearchParams, create_task

    hdr = FilterbankHeader(fch1=cfg["fch1"], foff=cfg["foff"], nchans=cfg["nchans"],
                           tsamp=cfg["tsamp"], nsamples=cfg["nsamples"])
    rfi = bool(cfg.get("rfi", False))
    params = SearchParams(dm_lo=cfg["dm_lo"], dm_hi=cfg["dm_hi"], spacing=LinearSpacing(cfg["dm_step"]),
                          engine=EngineConfig(n_workers=1, detect_thresh=cfg["detect_thresh"],
                                              boxcar_max=cfg["boxcar_max"]),
                          baseline_len_s=cfg["baseline_s"], nsamps_chunk=cfg["nsamps_chunk"],
                          rfi=RfiConfig(narrowband=rfi, broadband=rfi))
    return create_task(hdr, params)
