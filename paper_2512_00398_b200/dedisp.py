"""DM-trial plan: pulsegrid's dedisp.hpp host API (delay model and trial grid).

Mirrors /root/reference/proj/include/pulsegrid/dedisp.hpp:13-76 and
src/dedisp.cpp:13-74.  The arithmetic runs in libpgb200 (C++ compiled with the
reference build's FMA contractions spelled out), so delays are bit-identical to
the reference library's.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import abi
from ._native import check, lib

K_DISPERSION = 4.148808e3  # dedisp.hpp:13


@dataclass
class FilterbankHeader:
    """The fields of pulsegrid::FilterbankHeader (filterbank.hpp:22-43) the path uses."""

    fch1: float
    foff: float
    nchans: int
    tsamp: float
    nbits: int = 8
    nsamples: int = 0
    source_name: str = ""
    tstart: float = 0.0

    def channel_freq(self, channel: int) -> float:
        return self.fch1 + self.foff * channel

    def _c(self) -> abi.HeaderC:
        return abi.HeaderC(float(self.fch1), float(self.foff), float(self.tsamp), int(self.nchans), 0)


@dataclass
class LinearSpacing:
    step: float


@dataclass
class AdaptiveSpacing:
    tol: float


@dataclass
class DmTrialPlan:
    """pulsegrid::DmTrialPlan (dedisp.hpp:17-25): dms[ntrials], delays[ntrials][nchans]."""

    dms: np.ndarray
    delays: np.ndarray
    max_delay: int = field(init=False)

    def __post_init__(self):
        self.dms = np.ascontiguousarray(self.dms, np.float64)
        self.delays = np.ascontiguousarray(self.delays, np.int64)
        if self.delays.ndim != 2 or self.delays.shape[0] != self.dms.shape[0]:
            raise ValueError("delays must be [ntrials][nchans]")
        self.max_delay = int(self.delays.max()) if self.delays.size else 0

    @property
    def ntrials(self) -> int:
        return int(self.dms.shape[0])

    @property
    def nchans(self) -> int:
        return int(self.delays.shape[1])

    def trial_max_delay(self, trial: int) -> int:
        return int(self.delays[trial].max())


def delay_samples(dm: float, header: FilterbankHeader, channel: int) -> int:
    """src/dedisp.cpp:13-18."""
    h = header._c()
    return int(lib.pgb_delay_samples(float(dm), ctypes.byref(h), int(channel)))


def adaptive_dm_step(tol: float, header: FilterbankHeader) -> float:
    """src/dedisp.cpp:20-26."""
    h = header._c()
    return float(lib.pgb_adaptive_dm_step(float(tol), ctypes.byref(h)))


def generate_dm_trials(dm_lo: float, dm_hi: float, header: FilterbankHeader,
                       spacing: LinearSpacing | AdaptiveSpacing) -> DmTrialPlan:
    """src/dedisp.cpp:28-70; raises InvalidRangeError like the reference."""
    h = header._c()
    if isinstance(spacing, LinearSpacing):
        kind, val = abi.SPACING_LINEAR, spacing.step
    else:
        kind, val = abi.SPACING_ADAPTIVE, spacing.tol
    n = ctypes.c_size_t(0)
    check(lib.pgb_generate_dm_trials(float(dm_lo), float(dm_hi), ctypes.byref(h), kind, float(val),
                                     None, None, 0, ctypes.byref(n)))
    dms = np.zeros(n.value, np.float64)
    delays = np.zeros((n.value, header.nchans), np.int64)
    check(lib.pgb_generate_dm_trials(float(dm_lo), float(dm_hi), ctypes.byref(h), kind, float(val),
                                     abi.ptr(dms), abi.ptr(delays), n.value, ctypes.byref(n)))
    return DmTrialPlan(dms, delays)


def max_delay(plan: DmTrialPlan) -> int:
    return plan.max_delay
