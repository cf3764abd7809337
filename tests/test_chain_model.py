"""The exact event-replay model of an RFI-masked output's fp32 channel sum
(tools/fp32_chain_model.py): integer segment sums merged with the
per-binade fraction rounding, flagged cells as single fp32 adds, equal bit for bit to the
sequential fp32 sum whenever the model reports exact (CPU only)."""
import numpy as np
import pytest

from tools.fp32_chain_model import F32, chain_events, chain_sequential, merge


def _case(rng, n, p_flag, lo=0, hi=256, first_big=False):
    cells = rng.integers(lo, hi, n).astype(np.float32)
    if first_big:
        cells[:4] = rng.integers(100, 256, 4)
    flagged = rng.random(n) < p_flag
    counts = rng.integers(1, 65, n)
    sums = rng.integers(0, 256 * 64, n)
    cells[flagged] = (sums[flagged] / counts[flagged]).astype(np.float32)  # local means
    return cells, flagged


@pytest.mark.parametrize("seed", range(40))
def test_model_equals_sequential_sum(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(64, 4096))
    cells, flagged = _case(rng, n, p_flag=float(rng.choice([0.001, 0.01, 0.05, 0.3])),
                           first_big=bool(seed % 2))
    got, ok = chain_events(cells, flagged)
    want = chain_sequential(cells)
    if ok:
        assert got.view(np.uint32) == want.view(np.uint32), (seed, got, want)


def test_merge_crossing_several_binades():
    """A fraction carried through many binade crossings in one integer stretch."""
    rng = np.random.default_rng(7)
    checked = naive_wrong = 0
    for _ in range(3000):
        s = F32(rng.uniform(256, 4096))
        cells = rng.integers(0, 256, int(rng.integers(1, 2000))).astype(np.float32)
        want = F32(s)
        for x in cells:
            want = F32(want + x)
        got, ok = merge(s, int(cells.sum()))
        assert ok
        assert got.view(np.uint32) == want.view(np.uint32), (s, len(cells))
        naive_wrong += F32(s + F32(int(cells.sum()))).view(np.uint32) != want.view(np.uint32)
        checked += 1
    assert checked == 3000
    assert naive_wrong > 100  # one fp32 add of the stretch's sum is wrong in ~14 % of these


def test_small_state_is_reported():
    """Below 256 a single cell can skip a binade: merge must not claim exactness there."""
    s = F32(100.3)
    got, ok = merge(s, 300)
    assert not ok


def test_all_flagged_low_dm_output():
    """An output on a flagged row at DM 0 sees a flagged cell in every channel."""
    rng = np.random.default_rng(3)
    cells = (rng.integers(0, 256 * 64, 2048) / rng.integers(1, 65, 2048)).astype(np.float32)
    got, ok = chain_events(cells, np.ones(cells.size, bool))
    assert ok and got.view(np.uint32) == chain_sequential(cells).view(np.uint32)
