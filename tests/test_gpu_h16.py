"""RFI-masked 8-bit chunks on the device (SURVEY.md section 8 rows a3 + f1): the masked
integer path (zero replacement, bad channels only: the transpose zeroes the cells), the
widened-float fp32 path (local-mean rows, the default), and the fp16 in-order kernel with
exception rows (ablation library, PGB_RFI_H16=1) with its fp32 fallback.

Oracle: the reference library's own apply_mask (src/rfi.cpp:93-139) and run_dm_loop on the
masked float chunk (parity mode, src/engine.cpp:85-265); candidates compared field by
field with snr exact."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import ChunkSpec, Engine, EngineConfig, RfiConfig
from tests.helpers import FIELDS, assert_same_candidates, cfg_dict, u8_chunk

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _case(L, nch, dm_hi, dm_step, burst_every, seed, burst_rows=2, foff=-1.0):
    hdr = FilterbankHeader(fch1=1500.0, foff=foff, nchans=nch, tsamp=64e-6)
    plan = generate_dm_trials(0.0, dm_hi, hdr, LinearSpacing(dm_step))
    nt = plan.ntrials
    pulses = [(nt // 3, L // 5, 4, 30.0), (2 * nt // 3, L // 2, 16, 25.0)]
    data = u8_chunk(hdr, plan, L, seed, pulses=pulses).astype(np.int16)
    rng = np.random.default_rng(seed + 1)
    data[:, rng.choice(nch, max(1, nch // 20), replace=False)] += 40  # hot channels
    if burst_every:
        for t in range(burst_every // 2, L - burst_rows, burst_every):
            data[t: t + burst_rows, :] += 30  # DM-0 bursts (flagged rows)
    return hdr, plan, np.clip(data, 0, 255).astype(np.uint8)


def _cfg(hdr, boxcar_max=256, window=2001):
    return EngineConfig(n_workers=1, tsamp=hdr.tsamp, detect_thresh=6.0, boxcar_max=boxcar_max,
                        baseline_window=window)


def _order(c):
    return c[np.lexsort((c["width_index"], c["dm_trial"], c["peak_sample"]))]


def _check(engine, ref, hdr, plan, data, rfi, *, eng=None):
    L = data.shape[0]
    spec = ChunkSpec.whole(L)
    cfg = _cfg(hdr)
    masked, bc, bs = ref.rfi(data.astype(np.float32), narrowband=rfi.narrowband, broadband=rfi.broadband,
                             local_mean=rfi.local_mean)
    want, want_sk, _ = ref.run_dm_loop(masked, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    e = eng or engine
    got, _, skipped = e.search_file(data, L, [spec], plan, cfg, rfi=rfi)
    assert len(want) > 0
    assert_same_candidates(_order(got), _order(want))
    assert sorted(int(t) for _, t in np.asarray(skipped, np.uint64).reshape(-1, 2)) == sorted(int(t) for t in want_sk)
    return bc, bs


# E-like density: 2 flagged rows every 400 (a few per staged window), wide and narrow
# delay spreads, partial channel groups (nch % 8 != 0), one 8-channel stage of several
@pytest.mark.parametrize("L,nch,dm_hi,dm_step,every", [
    (20000, 256, 300.0, 2.0, 400),
    (12000, 100, 120.0, 4.0, 400),
    (30000, 512, 600.0, 3.0, 1000),
    (9000, 64, 40.0, 1.0, 250),
])
@pytest.mark.parametrize("kernel", [None, "PGB_RFI_H16", "PGB_RFI_HYB"])
def test_local_mean_matches_reference(engine, abl_engine, ref, monkeypatch, L, nch, dm_hi, dm_step, every, kernel):
    """Product (widened fp32 ring), the fp16 kernel and the event-replay kernel (ablation
    library) against the reference's masked chunk through run_dm_loop."""
    hdr, plan, data = _case(L, nch, dm_hi, dm_step, every, seed=L + nch)
    if kernel:
        monkeypatch.setenv(kernel, "1")
    bc, bs = _check(engine, ref, hdr, plan, data, RfiConfig(), eng=abl_engine if kernel else None)
    assert bc.any() and bs.any()


def test_dense_flags_take_the_float_fallback(abl_engine, ref, monkeypatch):
    """Bursts every 24 rows put more than HX_CAP (16) flagged rows in a staged window: the
    fp16 kernel hands the chunk to the widened-float fp32 path, same result."""
    hdr, plan, data = _case(12000, 128, 200.0, 2.0, 24, seed=77)
    monkeypatch.setenv("PGB_RFI_H16", "1")
    _, bs = _check(None, ref, hdr, plan, data, RfiConfig(), eng=abl_engine)
    assert bs.sum() > 16 * 10


@pytest.mark.parametrize("nch", [192, 100])  # 100: partial 64-channel tiles, rows not 16-byte multiples
@pytest.mark.parametrize("narrow,broad,local_mean", [(True, True, False), (True, False, True),
                                                     (False, True, False)])
def test_integer_masks_take_the_u8_path(engine, ref, narrow, broad, local_mean, nch):
    """Zero replacement or bad channels only: every cell stays an integer, the transpose zeroes
    the masked cells and the integer kernel runs."""
    hdr, plan, data = _case(16000, nch, 250.0, 2.0, 500, seed=5)
    _check(engine, ref, hdr, plan, data, RfiConfig(narrowband=narrow, broadband=broad, local_mean=local_mean))


def test_h16_equals_float_path(engine, abl_engine, monkeypatch):
    """The fp16 kernel (PGB_RFI_H16=1, ablation library) and the product's widened-float
    fp32 path produce identical candidates on a multi-chunk file with RFI excision."""
    hdr, plan, data = _case(3 * 8192, 256, 200.0, 2.0, 400, seed=9)
    L = data.shape[0]
    chunks = [ChunkSpec(index=i, start_sample=s, length=min(12000, L - s), overlap=0,
                        valid_begin=s, valid_end=min(s + 12000, L)) for i, s in enumerate(range(0, L, 12000))]
    cfg = _cfg(hdr)
    a = engine.search_file(data, L, chunks, plan, cfg, rfi=RfiConfig())
    monkeypatch.setenv("PGB_RFI_H16", "1")
    b = abl_engine.search_file(data, L, chunks, plan, cfg, rfi=RfiConfig())
    assert len(a[0]) > 0
    for k in FIELDS:
        assert np.array_equal(a[0][k], b[0][k]), k
    assert len(a[1]) == len(b[1])


WHICH = """
import sys; sys.path.insert(0, {root!r})
import numpy as np
from tests.test_gpu_h16 import _case, _cfg
from paper_2512_00398_b200.engine import ChunkSpec, Engine, RfiConfig
with Engine(0, ablations=True) as e:
    for every in (400, 24):
        hdr, plan, data = _case(12000, 128, 200.0, 2.0, every, seed=77)
        L = data.shape[0]
        e.search_file(data, L, [ChunkSpec.whole(L)], plan, _cfg(hdr), rfi=RfiConfig())
        print("done", every, file=sys.stderr, flush=True)
print("ok")
"""


def test_kernel_choice_h16_then_fallback():
    """PGB_DD_WHICH logs the kernel: with PGB_RFI_H16=1, E-like flags run the fp16 ring and
    dense flags fall back to the fp32 ring."""
    e = dict(os.environ, PGB_DD_WHICH="1", PGB_RFI_H16="1")
    out = subprocess.run([sys.executable, "-c", WHICH.format(root=str(ROOT))], env=e, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
    runs, cur = [], []
    for ln in out.stderr.splitlines():
        if ln.startswith("pgb dedisp:"):
            cur.append(ln.split()[2])
        elif ln.startswith("done"):
            runs.append(cur)
            cur = []
    assert len(runs) == 2, out.stderr[-2000:]
    assert "h16-ring" in runs[0] and "f32-ring" not in runs[0], runs
    assert "f32-ring" in runs[1] and "h16-ring" not in runs[1], runs
