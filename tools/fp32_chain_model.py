"""Host model of the exact event-replay formulation for RFI-masked chunks (DESIGN.md section
12, config E): an output's in-order fp32 channel sum (the reference's run_dm_loop,
src/dedisp.cpp:146-160) recomputed from integer segment sums and the flagged cells alone.

The chain s_{c+1} = fl32(s_c + x_c) over cells x_c >= 0 that are 8-bit integers except at a
few flagged channels (local-mean floats) equals:

  * between two flagged cells, a stretch of integer cells with integer sum n maps the state
    s to merge(s, n): fl32(s + n) when s is an integer or at most one binade is crossed,
    otherwise (s + n) with the fraction of s rounded to the ulp of every binade crossed, in
    order (round-to-nearest-even to a grid g <= 1/2 commutes with adding integers).  This
    needs s >= 256 (or an integral s): below 256 one cell can jump over a whole binade and
    the crossings are not determined by n alone -- `merge` reports that case;
  * a flagged cell v is one fp32 add fl32(s + v).

Not part of the product path; tests/test_chain_model.py checks it against the sequential
fp32 sum.  Valid while every partial sum stays below 2^21 (nchans * 255 < 2^21)."""
from __future__ import annotations

import numpy as np

F32 = np.float32


def _f(x) -> np.float32:
    return F32(x)


def merge(s: np.float32, n: int) -> tuple[np.float32, bool]:
    """State after integer cells summing to n >= 0 following state s >= 0; (value, exact).
    exact is False only when s < 256 is not an integer and two or more binades are crossed."""
    s = _f(s)
    if n == 0:
        return s, True
    r = _f(s + _f(n))
    if s == np.floor(s):
        return r, True
    es = int(np.frexp(s)[1])
    er = int(np.frexp(r)[1])
    if er - es <= 1:
        return r, True
    if s < 256:
        return r, False
    a = _f(np.floor(s))
    frac = _f(s - a)        # exact
    whole = _f(a + _f(n))   # exact integer (< 2^24)
    e = es                  # binade [2^(e-1), 2^e) holds s (frexp convention)
    while True:
        lo = float(2.0 ** e)  # the next binade boundary
        if float(whole) + float(frac) < lo:
            break
        m = _f(1.5 * lo)     # ulp(m) is the ulp of the binade [lo, 2 lo)
        frac = _f(_f(frac + m) - m)
        e += 1
    return _f(whole + frac), True


def chain_events(cells: np.ndarray, flagged: np.ndarray) -> tuple[np.float32, bool]:
    """cells: float32 values in channel order (integers except at `flagged`); the exact fp32
    chain from +0 rebuilt from integer segment sums and the flagged values."""
    s = _f(0.0)
    ok = True
    seg = 0
    for x, fl in zip(cells, flagged):
        if fl:
            s, good = merge(s, seg)
            ok &= good
            seg = 0
            s = _f(s + _f(x))
        else:
            seg += int(x)
    s, good = merge(s, seg)
    return s, ok & good


def chain_sequential(cells: np.ndarray) -> np.float32:
    s = _f(0.0)
    for x in cells:
        s = _f(s + _f(x))
    return s
