"""Full-size checks at BASELINE.json shapes, where the CPU oracle cannot run everything:
sampled trials of a config-B chunk are compared bit for bit with the naive definition,
and the whole-chunk candidate list is checked for the invariants the reference
guarantees (order, uniqueness, valid range, widths, recovery of every injected pulse)."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def config_b_chunk():
    import torch

    import bench

    cfg = dict(bench.CONFIG_B)
    task = bench.build_task(cfg)
    spec = task.chunks[0]
    payload = bench.make_payload(cfg, task.plan, rows=spec.length)
    torch.cuda.synchronize()
    return cfg, task, spec, payload


def test_config_b_sampled_trials_bit_exact(engine, port, config_b_chunk):
    cfg, task, spec, payload = config_b_chunk
    data = payload.cpu().numpy()
    plan = task.plan
    got = engine.dedisperse(data, plan, range(0, plan.ntrials))
    f = data.astype(np.float32)
    for t in (0, 517, plan.ntrials - 1):
        assert np.array_equal(got[t], port.dedisperse(f, plan.delays[t])), t


def test_config_b_chunk_invariants(engine, config_b_chunk):
    import bench
    from paper_2512_00398_b200.engine import Chunk

    cfg, task, spec, payload = config_b_chunk
    res = engine.run_dm_loop(Chunk(spec, payload), task.plan, task.engine)
    c = res.candidates
    assert len(c) > 0
    keys = np.stack([c["peak_sample"], c["dm_trial"], c["width_index"]]).T
    assert all(tuple(a) < tuple(b) for a, b in zip(keys[:-1], keys[1:]))  # strictly sorted, unique
    assert np.all((c["peak_sample"] >= spec.valid_begin) & (c["peak_sample"] < spec.valid_end))
    assert np.all(c["width_samples"] == (1 << c["width_index"].astype(np.uint64)))
    assert np.all(c["snr"] > cfg["detect_thresh"])
    assert np.all(c["begin_sample"] <= c["peak_sample"]) and np.all(c["peak_sample"] <= c["end_sample"])
    # every injected pulse inside chunk 0's valid range is recovered near its trial and time
    checked = 0
    for trial, t0, width, snr in bench.pulse_specs(cfg, task.plan):
        if not (spec.valid_begin <= t0 < spec.valid_end - 4096):
            continue
        if snr * 16.0 / np.sqrt(cfg["nchans"] * width) < 0.5:
            continue  # make_payload's round-half-up quantisation leaves this pulse out of the data
        checked += 1
        near = c[(np.abs(c["dm_trial"].astype(np.int64) - trial) <= 2) &
                 (np.abs(c["peak_sample"].astype(np.int64) - t0) <= width + 8)]
        assert len(near) > 0, (trial, t0, width, snr)
    assert checked > 0


def test_config_b_whole_file_recovers_pulses(engine):
    """All four chunks of config B through search_file: every injected pulse that survived
    quantisation is the representative of a cluster near its trial and time."""
    import bench

    cfg = dict(bench.CONFIG_B)
    task = bench.build_task(cfg)
    payload = bench.make_payload(cfg, task.plan)
    cands, clusters, skipped = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine)
    assert len(skipped) == 0 and len(cands) >= len(clusters.records)
    rep = clusters.representatives
    checked = 0
    for trial, t0, width, snr in bench.pulse_specs(cfg, task.plan):
        if snr * 16.0 / np.sqrt(cfg["nchans"] * width) < 0.5:
            continue
        checked += 1
        near = rep[(np.abs(rep["dm_trial"].astype(np.int64) - trial) <= 4) &
                   (np.abs(rep["peak_sample"].astype(np.int64) - t0) <= width + 8)]
        assert len(near) > 0, (trial, t0, width, snr)
    assert checked >= 5


def test_config_b_overlap_reuse_is_exact(engine, abl_engine, monkeypatch):
    """search_file moves the outputs chunk k-1 already dedispersed into chunk k instead of
    summing them again; the candidate list must equal the recompute-everything run."""
    import bench

    cfg = dict(bench.CONFIG_B)
    task = bench.build_task(cfg)
    payload = bench.make_payload(cfg, task.plan)
    a, ca, _ = engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine)
    _, _, adds_reuse = engine.last_dedisp_time()
    monkeypatch.setenv("PGB_NO_OVERLAP_REUSE", "1")
    b, cb, _ = abl_engine.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine)
    _, _, adds_full = abl_engine.last_dedisp_time()
    assert adds_reuse < 0.96 * adds_full  # the reuse actually happened
    assert len(a) == len(b) > 0
    for k in a.dtype.names:
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(ca.records, cb.records)
