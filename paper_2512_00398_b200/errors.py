"""Exception hierarchy mirroring pulsegrid's (/root/reference/proj/include/pulsegrid/errors.hpp:10-67).

The C ABI returns a status code naming the reference exception type; `raise_for`
rethrows it as the matching class so callers catch the same names they catch
around the reference library.
"""
from __future__ import annotations


class PulsegridError(RuntimeError):
    """pulsegrid::error (errors.hpp:10-12)."""


class ConfigError(PulsegridError):
    """pulsegrid::config_error (errors.hpp:65-67)."""


class InvalidRangeError(PulsegridError):
    """pulsegrid::invalid_range_error (errors.hpp:48-50)."""


class ChunkTooShortError(PulsegridError):
    """pulsegrid::chunk_too_short_error (errors.hpp:51-56); carries the trial index."""

    def __init__(self, msg: str, trial_index: int | None = None):
        super().__init__(msg)
        self.trial_index = trial_index


class BudgetExhaustedError(PulsegridError):
    """pulsegrid::budget_exhausted_error (errors.hpp:59-61)."""


class DegenerateSeriesError(PulsegridError):
    """pulsegrid::degenerate_series_error (errors.hpp:44-46)."""


class InvalidPlanError(PulsegridError):
    """pulsegrid::invalid_plan_error (errors.hpp:24-26)."""


class InsufficientStatisticsError(PulsegridError):
    """pulsegrid::insufficient_statistics_error (errors.hpp:40-42)."""


class ReadError(PulsegridError):
    """pulsegrid::read_error (errors.hpp:29-34): a chunk of the file could not be read."""


class DeviceError(PulsegridError):
    """No usable sm_100 device, a CUDA failure, or device OOM (no CPU fallback exists)."""


_BY_CODE = {
    1: ConfigError,
    2: InvalidRangeError,
    3: ChunkTooShortError,
    4: BudgetExhaustedError,
    5: DegenerateSeriesError,
    6: InvalidPlanError,
    7: ValueError,
    8: InsufficientStatisticsError,
    9: ReadError,
    100: DeviceError,
    101: DeviceError,
    102: DeviceError,
}


def raise_for(code: int, msg: str) -> None:
    if code == 0:
        return
    cls = _BY_CODE.get(code, PulsegridError)
    if cls is ChunkTooShortError:
        trial = None
        if msg.startswith("trial "):
            try:
                trial = int(msg.split()[1].rstrip(":"))
            except ValueError:
                trial = None
        raise ChunkTooShortError(msg, trial)
    raise cls(msg)
