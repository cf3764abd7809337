"""Every dedispersion kernel variant is bit-exact: the product library's default choice and
every PGB_* alternative of the ablation library (libpgb200_ablations.so; the switches are
read once per process, so each variant runs in its own interpreter) on a few of the
parity shapes (dedispersed sums against the C restatement of the naive definition)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SNIPPET = r'''
import os, sys
sys.path.insert(0, {root!r})
import numpy as np
from oracle.pyoracle import Port
from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing, generate_dm_trials
from paper_2512_00398_b200.engine import Engine
from tests.helpers import u8_chunk, f32_chunk
port = Port()
cases = [(4096, 1518.0, -0.0703125, 24000, 800.0, 8.0), (1024, 1500.0, -0.25, 20000, 500.0, 2.0),
         (517, 1450.0, -0.5, 12000, 400.0, 2.5)]
with Engine(0, ablations=bool(os.environ.get("PG_TEST_ABLATIONS"))) as eng:
    for nch, fch1, foff, L, dm_hi, step in cases:
        hdr = FilterbankHeader(fch1=fch1, foff=foff, nchans=nch, tsamp=64e-6)
        plan = generate_dm_trials(0.0, dm_hi, hdr, LinearSpacing(step))
        for data in (u8_chunk(hdr, plan, L, seed=nch), f32_chunk(nch, L, seed=nch, scale=5.0)):
            ok = [t for t in range(plan.ntrials) if plan.trial_max_delay(t) < L]
            got = eng.dedisperse(data, plan, range(0, len(ok)))
            for t in ok[::max(1, len(ok) // 6)] + [ok[-1]]:
                want = port.dedisperse(data.astype(np.float32) if data.dtype == np.uint8 else data,
                                       plan.delays[t])
                assert np.array_equal(got[t], want), (nch, t)
print("ok")
'''


@pytest.mark.parametrize("env", [
    {},                                   # persistent ring (u8, channel-paired K/T accumulation), fp32 ring
    {"PGB_DD_PERSIST0": "1"},             # grid-launched ring
    {"PGB_DD_RING": "0"},                 # CTA-barrier table kernel
    {"PGB_DD_RING2_OFF": "1"},            # wide windows: barrier kernel instead of the 2-slot ring
    {"PGB_RING_MODE": "2"},               # ring with IMAD addressing
    {"PGB_RING_MODE": "0"},               # persistent ring, every word accumulated as (LOP3, IMAD, LEA.HI)
    {"PGB_RING_MODE": "4"},               # odd words as (PRMT, IMAD, IMAD), even words as mode 0
    {"PGB_RING_MODE": "24"},              # channel pairs, T by IADD3 on even words
    {"PGB_F32_RING0": "1"},               # fp32 two-barrier kernel
    # mbarrier-ring race stress: random per-warp sleeps around the full / empty handshakes
    # scramble the warps' arrival order (racecheck does not model mbarrier acquire/release)
    {"PGB_RING_JITTER": "1"},
    {"PGB_RING_JITTER": "987654321"},
    {"PGB_RING_JITTER": "5", "PGB_DD_PERSIST0": "1"},
    {"PGB_DD_WARPS": "32"},               # 1024-thread ring, one trial per warp
    {"PGB_DD_WARPS": "32", "PGB_RING_JITTER": "3"},
])
def test_dedispersion_variants_bit_exact(env):
    e = dict(os.environ, **env)
    if env:
        e["PG_TEST_ABLATIONS"] = "1"
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(root=str(ROOT))], env=e,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


WIDE = SNIPPET.replace(
    "cases = [(4096, 1518.0, -0.0703125, 24000, 800.0, 8.0), (1024, 1500.0, -0.25, 20000, 500.0, 2.0),\n"
    "         (517, 1450.0, -0.5, 12000, 400.0, 2.5)]",
    "cases = [(4096, 1518.0, -0.0703125, 20000, 400.0, 4.0), (4096, 1518.0, -0.0703125, 16000, 300.0, 3.0),\n"
    "         (1024, 1500.0, -0.25, 20000, 500.0, 2.0)]")


@pytest.mark.parametrize("mode", ["", "0"])
def test_default_selection_covers_both_ring_depths(mode):
    """The default launcher picks the 3-slot ring for narrow windows and the 2-slot ring when
    three slots would force narrower stages; both bit-exact (PGB_DD_WHICH logs the choice),
    with the default and the per-word (mode 0) accumulation."""
    assert WIDE != SNIPPET
    e = dict(os.environ, PGB_DD_WHICH="1")
    if mode:
        e["PGB_RING_MODE"] = mode
        e["PG_TEST_ABLATIONS"] = "1"
    out = subprocess.run([sys.executable, "-c", WIDE.format(root=str(ROOT))], env=e,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
    kinds = {line.split()[2] for line in out.stderr.splitlines() if line.startswith("pgb dedisp:")}
    assert "ring3-persist" in kinds and "ring2-persist" in kinds, kinds
