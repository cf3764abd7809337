"""Host logic around the path: chunk plan, task resolution, SIGPROC ingest, .cand text."""
import numpy as np
import pytest

from paper_2512_00398_b200 import abi, errors
from paper_2512_00398_b200.cluster import Clusters
from paper_2512_00398_b200.dedisp import LinearSpacing
from paper_2512_00398_b200.engine import EngineConfig
from paper_2512_00398_b200.pipeline import (SearchParams, baseline_window_samples, create_task,
                                            plan_chunks, read_filterbank, write_candidates)

from .helpers import random_candidates


def test_plan_chunks_examples():
    # SPEC.md plan_chunks examples; src/filterbank.cpp:239-272
    p = plan_chunks(1000, 400, 100)
    assert [c.start_sample for c in p] == [0, 300, 600]
    assert [(c.valid_begin, c.valid_end) for c in p] == [(0, 300), (300, 600), (600, 1000)]
    p = plan_chunks(500, 800, 100)
    assert len(p) == 1 and p[0].length == 500 and p[0].overlap == 0
    with pytest.raises(errors.InvalidPlanError):
        plan_chunks(1000, 100, 100)


@pytest.mark.parametrize("args", [(10000, 1024, 200), (2 ** 20, 2 ** 18, 33519), (937500, 32768, 2646),
                                  (12345, 12346, 10)])
def test_plan_chunks_vs_reference(ref, args):
    want = ref.plan_chunks(*args)
    got = plan_chunks(*args)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g.index, g.start_sample, g.length, g.overlap, g.valid_begin, g.valid_end) == tuple(
            int(w[k]) for k in ("index", "start_sample", "length", "overlap", "valid_begin", "valid_end"))
    # valid ranges tile [0, nsamples)
    assert got[0].valid_begin == 0 and got[-1].valid_end == args[0]
    assert all(a.valid_end == b.valid_begin for a, b in zip(got, got[1:]))


def test_create_task_and_ingest_match_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    nch, n = 64, 20000
    grid = np.floor(rng.normal(100, 16, (n, nch)) + 0.5).clip(0, 255).astype(np.float32)
    path = tmp_path / "t.fil"
    ref.write_filterbank(path, grid, 1500.0, -2.0, 64e-6, nbits=8)
    hdr, payload = read_filterbank(path)
    assert hdr.nchans == nch and hdr.nsamples == n and hdr.tsamp == 64e-6
    assert np.array_equal(payload, grid.astype(np.uint8))
    params = SearchParams(dm_lo=0.0, dm_hi=150.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=256), baseline_len_s=0.1, nsamps_chunk=8192)
    task = create_task(hdr, params)
    want, bw = ref.create_task_plan(path, dm_lo=0.0, dm_hi=150.0, dm_step=2.0, boxcar_max=256,
                                    baseline_len_s=0.1, nsamps_chunk=8192)
    assert task.engine.baseline_window == bw == baseline_window_samples(0.1, 64e-6)
    assert [(c.start_sample, c.length, c.overlap) for c in task.chunks] == [
        (int(w["start_sample"]), int(w["length"]), int(w["overlap"])) for w in want]


def test_write_candidates_matches_reference(ref, port):
    rng = np.random.default_rng(9)
    cands = random_candidates(rng, 300, 20000)
    recs, members = port.link_grid(cands, (3, 9, 3))
    text = write_candidates(Clusters(recs, members))
    assert text == ref.write_candidates(recs)
    assert text == port.format_candidates(recs)


def test_baseline_window_rounding():
    assert baseline_window_samples(2.0, 64e-6) == 31251
    assert baseline_window_samples(2.0, 49.152e-6) == 40691
    assert baseline_window_samples(0.0, 64e-6) == 0
    assert baseline_window_samples(1e-9, 64e-6) == 1


def test_host_pack_u8_round_trip(tmp_path):
    """The drop-in's host repack of widened 8-bit chunks (csrc/host_pack.cpp, AVX2 + scalar):
    exact bytes for integral cells, failure for any other cell (tests/cpp/host_pack_check.cpp)."""
    import shutil
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    src = root / "paper_2512_00398_b200" / "csrc" / "host_pack.cpp"
    if not shutil.which("g++"):
        pytest.skip("no g++")
    exe = tmp_path / "pack_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", str(root / "tests" / "cpp" / "host_pack_check.cpp"),
                    str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "pack ok" in out.stdout, out.stdout + out.stderr
