"""Drop-in proof by link substitution and file-level parity.

The reference's own create_task + execute_task (src/pipeline.cpp:32-119) runs twice
on the same SIGPROC file: once fully reference (oracle/_ref/pipeline_ref) and once
with the engine/cluster objects replaced by paper_2512_00398_b200/dropin over
libpgb200 (oracle/_ref/pipeline_b200).  The .cand files must be byte-identical.
The Python product path (pipeline.search_file + write_candidates) must produce the
same bytes too.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import LinearSpacing
from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
from paper_2512_00398_b200.pipeline import SearchParams, create_task, read_filterbank, search_file, write_candidates

pytestmark = pytest.mark.gpu

REF_DIR = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _need_binaries():
    for b in ("pipeline_ref", "pipeline_b200"):
        if not (REF_DIR / b).exists():
            pytest.skip(f"{b} not built (make -C oracle dropin)")


def _u8_file(ref, path, nch=256, n=1 << 17, seed=11):
    fch1, foff, tsamp = 1500.0, -1.0, 64e-6
    rng = np.random.default_rng(seed)
    grid = rng.normal(100.0, 16.0, (n, nch)).astype(np.float32)
    for dm, t0, w, snr in [(60.0, 20000, 4, 20.0), (150.0, 61000, 16, 16.0), (240.0, 101000, 64, 25.0)]:
        ref.inject_pulse(grid, fch1, foff, tsamp, dm, t0 * tsamp, w, ref.amplitude_for_snr(snr, 16.0, nch, w))
    ref.write_filterbank(path, grid, fch1, foff, tsamp, nbits=8)


def _run(binary, fil, cand, args):
    out = subprocess.run([str(REF_DIR / binary), str(fil), str(cand), *map(str, args)],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


ARGS_U8 = (0.0, 300.0, 2.0, 1024, 0.5, 1 << 15, 16)  # dm_lo dm_hi step boxcar baseline_s chunk workers


def test_link_substitution_u8(ref, tmp_path):
    _need_binaries()
    fil = tmp_path / "u8.fil"
    _u8_file(ref, fil)
    a = _run("pipeline_ref", fil, tmp_path / "ref.cand", ARGS_U8)
    b = _run("pipeline_b200", fil, tmp_path / "b200.cand", ARGS_U8)
    assert a["chunks"] > 1 and a["clusters"] > 0
    ref_text = (tmp_path / "ref.cand").read_text()
    assert (tmp_path / "b200.cand").read_text() == ref_text
    assert a["clusters"] == b["clusters"] and a["skipped"] == b["skipped"]
    # and the Python product path over raw u8 ingest gives the same bytes
    hdr, payload = read_filterbank(fil)
    params = SearchParams(dm_lo=ARGS_U8[0], dm_hi=ARGS_U8[1], spacing=LinearSpacing(ARGS_U8[2]),
                          engine=EngineConfig(boxcar_max=ARGS_U8[3]), baseline_len_s=ARGS_U8[4],
                          nsamps_chunk=ARGS_U8[5], rfi=RfiConfig(False, False))
    res = search_file(payload, create_task(hdr, params))
    assert write_candidates(res.clusters) == ref_text


def test_timing_sink_records_processed_trials(ref, tmp_path, monkeypatch):
    """EngineConfig::timing_sink (engine.hpp:16-23): the drop-in emits one TrialTiming per
    trial that finished the chain in each chunk -- the same multiset of trial ids as the
    reference's execute_task -- with the device stage times amortised over them."""
    _need_binaries()
    fil = tmp_path / "u8.fil"
    _u8_file(ref, fil)
    recs = {}
    for binary in ("pipeline_ref", "pipeline_b200"):
        out = tmp_path / f"{binary}.timing"
        monkeypatch.setenv("PG_TIMING_OUT", str(out))
        _run(binary, fil, tmp_path / f"{binary}.cand", ARGS_U8)
        rows = [line.split() for line in out.read_text().splitlines()]
        recs[binary] = ([int(r[0]) for r in rows], [[float(v) for v in r[1:]] for r in rows])
    ref_trials, _ = recs["pipeline_ref"]
    b_trials, b_ms = recs["pipeline_b200"]
    assert len(ref_trials) > 0
    assert sorted(b_trials) == sorted(ref_trials)
    ms = np.asarray(b_ms)
    assert (ms >= 0).all() and (ms[:, 0] > 0).all() and (ms[:, 2] > 0).all() and (ms[:, 3] > 0).all()
    assert (ms[:, 1] > 0).all()  # baseline on (baseline_s = 0.5)


def test_link_substitution_f32_file(ref, tmp_path):
    """nbits=32 Gaussian file (tests/test_pipeline.cpp:24-35 style): the fp32 in-order path."""
    _need_binaries()
    nch, n, fch1, foff, tsamp = 16, 16384, 1500.0, -4.0, 64e-6
    grid = ref.generate_noise(fch1, foff, tsamp, nch, n, 0.0, 1.0, 5)
    ref.inject_pulse(grid, fch1, foff, tsamp, 60.0, 4000 * tsamp, 4, ref.amplitude_for_snr(18.0, 1.0, nch, 4))
    fil = tmp_path / "f32.fil"
    ref.write_filterbank(fil, grid, fch1, foff, tsamp, nbits=32)
    args = (0.0, 100.0, 2.0, 32, 0.05, 8192, 2)
    a = _run("pipeline_ref", fil, tmp_path / "ref.cand", args)
    b = _run("pipeline_b200", fil, tmp_path / "b200.cand", args)
    assert a["chunks"] > 1
    assert (tmp_path / "b200.cand").read_text() == (tmp_path / "ref.cand").read_text()
    assert a["clusters"] == b["clusters"] > 0


@pytest.mark.slow
def test_link_substitution_config_b_matches_golden(tmp_path):
    """The reference's own execute_task with our engine/cluster TUs linked in, on the full
    config-B file (5 chunks of read_chunk's widened floats, repacked to bytes on the host
    before the upload): .cand bytes equal the pure reference's (tests/golden/config_B.npz)."""
    import numpy as np

    from tests.helpers import task_for
    from tools import synth

    _need_binaries()
    z = np.load(Path(__file__).resolve().parent / "golden" / "config_B.npz")
    cfg = json.loads(str(z["meta"]))["cfg"]
    fil = tmp_path / "B.fil"
    synth.write_filterbank(fil, cfg, task_for(cfg).plan.delays)
    args = (cfg["dm_lo"], cfg["dm_hi"], cfg["dm_step"], cfg["boxcar_max"], cfg["baseline_s"], cfg["nsamps_chunk"], 16)
    b = _run("pipeline_b200", fil, tmp_path / "b200.cand", args)
    assert b["chunks"] == 5
    assert (tmp_path / "b200.cand").read_text() == z["cand_text"].tobytes().decode()
