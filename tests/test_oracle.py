"""The CPU oracles, pinned before they are trusted (no GPU needed).

* the C restatement (oracle/pg_oracle.c) reproduces the golden fixtures made from
  the compiled reference library (tests/golden/make_golden.py) and the reference
  unit tests' known answers;
* where the reference library is built (oracle/_ref), restatement == reference on
  fresh random cases, field by field;
* the shipped multi-trial dedispersion path of the reference is defective (SURVEY.md
  section 0), which is why every oracle runs in parity mode.
"""
from pathlib import Path

import numpy as np
import pytest

from .helpers import FIELDS, assert_same_candidates, random_candidates

GOLDEN = np.load(Path(__file__).parent / "golden" / "golden_ref.npz")


def test_known_answers(port):
    # tests/test_dedisp.cpp:16-30, :77-103, :116-129
    assert port.delay_samples(100.0, 1500.0, -1.0, 64e-6, 101, 100) == 426 == int(GOLDEN["delay_426"])
    _, d = port.generate_dm_trials(0.0, 1000.0, 1500.0, -1.0, 64e-6, 501, step=250.0)
    assert int(d.max()) == 36014 == int(GOLDEN["max_delay_36014"])
    dms, _ = port.generate_dm_trials(0.0, 1000.0, 1500.0, -1.0, 64e-6, 64, tol=1.25)
    assert len(dms) == 10328 == int(GOLDEN["adaptive_count_10328"])
    assert dms[-1] == 1000.0


def test_linear_spacing_and_ranges(port):
    # tests/test_dedisp.cpp:45-75
    dms, _ = port.generate_dm_trials(0.0, 10.0, 1500.0, -1.0, 64e-6, 8, step=2.5)
    assert np.allclose(dms, [0, 2.5, 5, 7.5, 10])
    dms, _ = port.generate_dm_trials(0.0, 9.0, 1500.0, -1.0, 64e-6, 8, step=2.5)
    assert len(dms) == 5 and dms[-1] == 9.0
    assert len(port.generate_dm_trials(5.0, 5.0, 1500.0, -1.0, 64e-6, 8, tol=1.25)[0]) == 1
    from oracle.pyoracle import OracleError

    for args in [dict(step=1.0, lo=10.0, hi=5.0), dict(step=0.0, lo=0.0, hi=10.0),
                 dict(tol=1.0, lo=0.0, hi=10.0)]:
        lo, hi = args.pop("lo"), args.pop("hi")
        with pytest.raises(OracleError):
            port.generate_dm_trials(lo, hi, 1500.0, -1.0, 64e-6, 8, **args)


def test_config_b_plan_matches_golden(port):
    dms, delays = port.generate_dm_trials(0.0, 2000.0, 1518.0, -0.0703125, 64e-6, 4096, step=2.0)
    assert np.array_equal(dms, GOLDEN["planB_dms"])
    assert int(delays.sum()) == int(GOLDEN["planB_delays_sum"])
    assert np.array_equal(delays[::100], GOLDEN["planB_delays_rows"])
    assert int(delays.max()) == 29423


def test_run_dm_loop_u8_golden(port):
    data = GOLDEN["u8_data"]
    spec = dict(index=0, start_sample=0, length=data.shape[0], overlap=0, valid_begin=0,
                valid_end=data.shape[0])
    cfg = dict(n_workers=4, tsamp=64e-6, detect_thresh=6.0, boxcar_max=256, baseline_window=2001)
    cands, skipped = port.run_dm_loop(data, spec, GOLDEN["u8_dms"], GOLDEN["u8_delays"], cfg)
    assert_same_candidates(cands, GOLDEN["u8_cands"])
    assert np.array_equal(skipped, GOLDEN["u8_skipped"])


def test_run_dm_loop_f32_golden(port):
    g = GOLDEN["f32_noise"]
    spec = dict(index=0, start_sample=0, length=8192, overlap=0, valid_begin=0, valid_end=8192)
    cfg = dict(n_workers=2, tsamp=64e-6, detect_thresh=6.0, boxcar_max=64, baseline_window=1001)
    cands, skipped = port.run_dm_loop(g, spec, GOLDEN["f32_dms"], GOLDEN["f32_delays"], cfg)
    assert_same_candidates(cands, GOLDEN["f32_cands"])
    assert np.array_equal(skipped, GOLDEN["f32_skipped"])


def test_link_grid_and_cand_text_golden(port):
    clusters, members = port.link_grid(GOLDEN["u8_cands"], (3, 9, 3))
    want = GOLDEN["u8_clusters"]
    assert len(clusters) == len(want)
    for k in FIELDS:
        assert np.array_equal(clusters["representative"][k], want["representative"][k]), k
    for k in ("members", "begin_sample", "end_sample", "dm_lo", "dm_hi"):
        assert np.array_equal(clusters[k], want[k]), k
    assert port.format_candidates(clusters) == GOLDEN["u8_cand_text"].tobytes().decode()


def test_cand_line_format(port):
    # tests/test_pipeline.cpp:71-77
    from paper_2512_00398_b200 import abi

    c = np.zeros(1, abi.CLUSTER_DTYPE)
    r = c["representative"]
    r["snr"], r["peak_sample"], r["time_s"] = 20.5, 1000, 1000 * 64e-6
    r["width_index"], r["dm_trial"], r["dm"] = 3, 42, 105.0
    c["members"], c["begin_sample"], c["end_sample"] = 7, 996, 1012
    assert port.format_candidates(c) == "20.50\t1000\t0.064000000\t3\t42\t105.000\t7\t996\t1012\n"


# ---- restatement vs the compiled reference (where built) ------------------------------

@pytest.mark.parametrize("cfgB", [(1024, 1500.0, -0.25, 500.0, 2.0), (4096, 1518.0, -0.0703125, 2000.0, 2.0),
                                  (4096, 1500.0, -0.1220703125, 5000.0, 1.25),
                                  (8192, 1500.0, -0.0625, 2047.5, 0.5)])
def test_plans_vs_reference(port, ref, cfgB):
    nch, fch1, foff, hi, step = cfgB
    tsamp = 49.152e-6 if hi == 5000.0 else 64e-6
    a = ref.generate_dm_trials(0.0, hi, fch1, foff, tsamp, nch, step=step)
    b = port.generate_dm_trials(0.0, hi, fch1, foff, tsamp, nch, step=step)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_run_dm_loop_vs_reference_random(port, ref, seed):
    rng = np.random.default_rng(seed)
    nch = int(rng.integers(8, 64))
    L = int(rng.integers(3000, 9000))
    foff = -float(rng.integers(1, 6))
    dms, delays = ref.generate_dm_trials(0.0, float(rng.integers(50, 200)), 1500.0, foff, 64e-6, nch,
                                         step=float(rng.integers(2, 9)))
    data = rng.normal(0.0, 1.0, (L, nch)).astype(np.float32)
    start = int(rng.integers(0, 2)) * 5000
    spec = dict(index=1, start_sample=start, length=L, overlap=int(rng.integers(0, 2)) * 300,
                valid_begin=start + 100, valid_end=start + L - 400)
    cfg = dict(n_workers=3, tsamp=64e-6, detect_thresh=float(rng.uniform(3.0, 5.0)),
               boxcar_max=int(2 ** rng.integers(0, 9)), baseline_window=int(rng.integers(0, 4000)))
    a, sa, _ = ref.run_dm_loop(data, spec, dms, delays, cfg)
    b, sb = port.run_dm_loop(data, spec, dms, delays, cfg)
    assert len(a) > 0
    assert_same_candidates(b, a)
    assert np.array_equal(sa, sb)


def test_link_grid_vs_reference_random(port, ref):
    rng = np.random.default_rng(31)
    for _ in range(40):
        n = int(rng.integers(1, 400))
        cands = random_candidates(rng, n, int(rng.integers(1, 50000)))
        radii = (int(rng.integers(1, 6)), int(rng.integers(0, 12)), int(rng.integers(0, 4)))
        a, am, _ = ref.link_grid(cands, radii)
        b, bm = port.link_grid(cands, radii)
        assert len(a) == len(b)
        for k in ("members", "begin_sample", "end_sample", "dm_lo", "dm_hi"):
            assert np.array_equal(a[k], b[k])
        assert np.array_equal(a["representative"]["peak_sample"], b["representative"]["peak_sample"])
        assert np.array_equal(a["representative"]["dm_trial"], b["representative"]["dm_trial"])
        # the quadratic reference clustering agrees too (tests/test_cluster.cpp:102-120)
        c, cm, _ = ref.link_grid(cands, radii, reference=True)
        assert np.array_equal(a["members"], c["members"])


def test_reference_block_path_defect(ref):
    """dedisperse_block with two trials over > 1 tile re-adds tails (src/dedisp.cpp:188-195):
    the reason every oracle here runs with block size 1 (parity mode)."""
    rng = np.random.default_rng(5)
    nch, L = 16, 9000
    dms, delays = ref.generate_dm_trials(0.0, 400.0, 1500.0, -8.0, 64e-6, nch, step=100.0)
    data = rng.integers(0, 10, (L, nch)).astype(np.float32)
    naive = [ref.dedisperse(data, dms, delays, t) for t in (1, 4)]
    block = ref.dedisperse_block(data, dms, delays, [1, 4])
    assert np.array_equal(block[0], naive[0]) or np.array_equal(block[1], naive[1])
    assert not (np.array_equal(block[0], naive[0]) and np.array_equal(block[1], naive[1]))


@pytest.mark.parametrize("name", ["A", "B", "C1", "E1"])
def test_restatement_reproduces_config_golden_clusters(port, name):
    """The C restatement's link_grid and .cand writer, on the reference pipeline's own
    full-size candidate lists (tests/golden/config_<name>.npz), give the reference's
    clusters, member ids and .cand text exactly."""
    import json
    from pathlib import Path

    gz = Path(__file__).resolve().parent / "golden" / f"config_{name}.npz"
    if not gz.exists():
        pytest.skip(f"{gz.name} not generated")
    z = np.load(gz)
    meta = json.loads(str(z["meta"]))
    assert "candidates" in z.files and len(z["candidates"]) == meta["ncandidates"]
    recs, members = port.link_grid(z["candidates"], (3, 9, 3))
    want = z["clusters"]
    assert len(recs) == len(want) == meta["nclusters"]
    for k in ("members", "begin_sample", "end_sample", "dm_lo", "dm_hi"):
        assert np.array_equal(recs[k], want[k]), k
    for k in ("peak_sample", "dm_trial", "width_index", "snr"):
        assert np.array_equal(recs["representative"][k], want["representative"][k]), k
    wm = z["members"]
    for i in range(len(want)):  # member ids per cluster (flat layouts may order clusters differently)
        a = members[int(recs["member_offset"][i]): int(recs["member_offset"][i]) + int(recs["members"][i])]
        b = wm[int(want["member_offset"][i]): int(want["member_offset"][i]) + int(want["members"][i])]
        assert np.array_equal(a, b), i
    assert port.format_candidates(recs) == z["cand_text"].tobytes().decode()


def test_config_a_generator_matches_golden_digest():
    """tools/synth.py regenerates the exact bytes the golden run searched (config A here;
    the GPU tests check the larger configs the same way)."""
    import hashlib
    import json
    from pathlib import Path

    from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
    from tools import synth

    z = np.load(Path(__file__).resolve().parent / "golden" / "config_A.npz")
    meta = json.loads(str(z["meta"]))
    cfg = meta["cfg"]
    hdr = FilterbankHeader(fch1=cfg["fch1"], foff=cfg["foff"], nchans=cfg["nchans"], tsamp=cfg["tsamp"])
    plan = generate_dm_trials(cfg["dm_lo"], cfg["dm_hi"], hdr, LinearSpacing(cfg["dm_step"]))
    assert hashlib.sha256(synth.payload(cfg, plan.delays).tobytes()).hexdigest() == meta["payload_sha256"]
