"""Device RFI excision against the reference's
flag_narrowband / flag_broadband / apply_mask, and the whole file search with RFI on."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2512_00398_b200 import errors
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Engine, EngineConfig, RfiConfig
from paper_2512_00398_b200.pipeline import SearchParams, create_task, read_filterbank, search_file, write_candidates

pytestmark = pytest.mark.gpu

REF_DIR = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def _plan(nch):
    hdr = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=nch, tsamp=64e-6)
    return generate_dm_trials(0.0, 10.0, hdr, LinearSpacing(5.0))


def _dirty_u8(L, nch, seed):
    """8-bit noise with hot channels, a noisy channel and DM-0 bursts every ~400 samples."""
    rng = np.random.default_rng(seed)
    x = rng.normal(100.0, 16.0, (L, nch))
    hot = rng.choice(nch, max(1, nch // 20), replace=False)
    x[:, hot] += 45.0
    x[:, (hot[0] + 1) % nch] += rng.normal(0, 60.0, L)
    for t in range(137, L - 3, 401):
        x[t: t + 2, :] += 50.0
    return np.clip(np.floor(x + 0.5), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("local_mean", [True, False])
# 16-byte rows take the integer-sum / staged-variance kernels (partial channel CTAs: 80,
# 1040; partial row stages: 20000, 700); 36 widens 4 cells a thread only; 13 is all scalar
@pytest.mark.parametrize("L,nch", [(4096, 64), (20000, 256), (3000, 13), (700, 80), (9000, 1040), (2500, 36)])
def test_rfi_clean_u8_matches_reference(engine, ref, L, nch, local_mean):
    data = _dirty_u8(L, nch, seed=L + nch)
    want, wbc, wbs = ref.rfi(data.astype(np.float32), local_mean=local_mean)
    got, gbc, gbs = engine.rfi_clean(data, _plan(nch), RfiConfig(local_mean=local_mean))
    assert np.array_equal(gbc, wbc) and np.array_equal(gbs, wbs)
    assert wbc.any() and wbs.any()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_rfi_scalar_kernels_agree(engine, ref, monkeypatch):
    """PGB_RFI_SERIAL=1 (one thread per channel / sample, separate bad-channel pass) and the
    default integer-sum kernels give identical flags and masked chunks."""
    data = _dirty_u8(5000, 96, seed=11)
    a = engine.rfi_clean(data, _plan(96), RfiConfig())
    monkeypatch.setenv("PGB_RFI_SERIAL", "1")
    with Engine(0, ablations=True) as abl:
        b = abl.rfi_clean(data, _plan(96), RfiConfig())
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_rfi_clean_f32_matches_reference(engine, ref):
    rng = np.random.default_rng(3)
    L, nch = 6000, 48
    x = rng.normal(0.0, 1.0, (L, nch)).astype(np.float32)
    x[:, 7] += 3.0
    x[2000:2003, :] += 4.0
    want, wbc, wbs = ref.rfi(x)
    got, gbc, gbs = engine.rfi_clean(x, _plan(nch), RfiConfig())
    assert np.array_equal(gbc, wbc) and np.array_equal(gbs, wbs)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("narrow,broad", [(True, False), (False, True)])
def test_rfi_single_flagger(engine, ref, narrow, broad):
    data = _dirty_u8(5000, 32, seed=9)
    want, wbc, wbs = ref.rfi(data.astype(np.float32), narrowband=narrow, broadband=broad)
    got, gbc, gbs = engine.rfi_clean(data, _plan(32), RfiConfig(narrowband=narrow, broadband=broad))
    assert np.array_equal(gbc, wbc) and np.array_equal(gbs, wbs)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_rfi_needs_four_channels(engine):
    # src/rfi.cpp:33-34
    with pytest.raises(errors.InsufficientStatisticsError):
        engine.rfi_clean(np.full((100, 3), 7, np.uint8), _plan(3), RfiConfig())


def _write_dirty_file(ref, path, nch=128, n=1 << 16):
    fch1, foff, tsamp = 1500.0, -2.0, 64e-6
    rng = np.random.default_rng(21)
    grid = rng.normal(100.0, 16.0, (n, nch)).astype(np.float32)
    for dm, t0, w, snr in [(50.0, 12000, 4, 25.0), (120.0, 40000, 16, 20.0)]:
        ref.inject_pulse(grid, fch1, foff, tsamp, dm, t0 * tsamp, w, ref.amplitude_for_snr(snr, 16.0, nch, w))
    grid[:, [3, 77]] += 40.0
    for t in range(500, n - 4, 4096):
        grid[t: t + 3, :] += 60.0
    ref.write_filterbank(path, grid, fch1, foff, tsamp, nbits=8)


def test_file_search_with_rfi_matches_reference(ref, tmp_path):
    """RFI on (reference defaults): the reference pipeline with the drop-in engine, and the
    Python path with device RFI + the fp32 dedispersion path, write the reference's bytes."""
    fil = tmp_path / "dirty.fil"
    _write_dirty_file(ref, fil)
    args = [str(fil), "", "0", "200", "2", "512", "0.5", str(1 << 15), "8", "1"]
    outs = {}
    for b in ("pipeline_ref", "pipeline_b200"):
        if not (REF_DIR / b).exists():
            pytest.skip("drop-in binaries not built")
        args[1] = str(tmp_path / f"{b}.cand")
        r = subprocess.run([str(REF_DIR / b), *args], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        outs[b] = json.loads(r.stdout)
    ref_text = (tmp_path / "pipeline_ref.cand").read_text()
    assert outs["pipeline_ref"]["clusters"] > 0
    assert (tmp_path / "pipeline_b200.cand").read_text() == ref_text
    hdr, payload = read_filterbank(fil)
    params = SearchParams(dm_lo=0.0, dm_hi=200.0, spacing=LinearSpacing(2.0),
                          engine=EngineConfig(boxcar_max=512), baseline_len_s=0.5,
                          nsamps_chunk=1 << 15, rfi=RfiConfig())
    res = search_file(payload, create_task(hdr, params))
    assert write_candidates(res.clusters) == ref_text
