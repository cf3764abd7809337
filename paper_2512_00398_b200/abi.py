"""Record layouts of the C ABI (include/pulsegrid_b200.h) as numpy dtypes / ctypes.

The candidate record is byte-for-byte pulsegrid::Candidate
(/root/reference/proj/include/pulsegrid/detect.hpp:14-25, 72 bytes) so arrays
cross the boundary without conversion.
"""
from __future__ import annotations

import ctypes

import numpy as np

CANDIDATE_DTYPE = np.dtype(
    {
        "names": ["snr", "peak_sample", "time_s", "width_index", "width_samples",
                  "dm_trial", "dm", "begin_sample", "end_sample"],
        "formats": ["<f4", "<u8", "<f8", "<u4", "<u8", "<u4", "<f8", "<u8", "<u8"],
        "offsets": [0, 8, 16, 24, 32, 40, 48, 56, 64],
        "itemsize": 72,
    }
)

CLUSTER_DTYPE = np.dtype(
    {
        "names": ["representative", "members", "begin_sample", "end_sample", "dm_lo", "dm_hi",
                  "member_offset"],
        "formats": [CANDIDATE_DTYPE, "<u8", "<u8", "<u8", "<f8", "<f8", "<u8"],
        "offsets": [0, 72, 80, 88, 96, 104, 112],
        "itemsize": 120,
    }
)

CHUNK_SPEC_DTYPE = np.dtype(
    [("index", "<u8"), ("start_sample", "<u8"), ("length", "<u8"), ("overlap", "<u8"),
     ("valid_begin", "<u8"), ("valid_end", "<u8")]
)

# status codes (pgb_status)
OK = 0
ERR_CONFIG = 1
ERR_INVALID_RANGE = 2
ERR_CHUNK_TOO_SHORT = 3
ERR_BUDGET = 4
ERR_DEGENERATE = 5
ERR_INVALID_PLAN = 6
ERR_ARGUMENT = 7
ERR_INSUFFICIENT = 8
ERR_NO_DEVICE = 100
ERR_CUDA = 101
ERR_OOM = 102

SPACING_LINEAR = 0
SPACING_ADAPTIVE = 1


class ChunkSpecC(ctypes.Structure):
    _fields_ = [("index", ctypes.c_uint64), ("start_sample", ctypes.c_uint64),
                ("length", ctypes.c_uint64), ("overlap", ctypes.c_uint64),
                ("valid_begin", ctypes.c_uint64), ("valid_end", ctypes.c_uint64)]


class EngineConfigC(ctypes.Structure):
    _fields_ = [("n_workers", ctypes.c_uint32), ("detect_thresh", ctypes.c_float),
                ("tsamp", ctypes.c_double), ("boxcar_max", ctypes.c_uint64),
                ("baseline_window", ctypes.c_uint64), ("memory_budget", ctypes.c_uint64),
                ("max_in_flight", ctypes.c_uint64)]


class LinkRadiiC(ctypes.Structure):
    _fields_ = [("sep_time", ctypes.c_uint64), ("sep_dm_trials", ctypes.c_uint32),
                ("sep_width", ctypes.c_uint32)]


class RfiConfigC(ctypes.Structure):
    _fields_ = [("narrowband", ctypes.c_int32), ("broadband", ctypes.c_int32),
                ("k_sigma", ctypes.c_double), ("k_mad", ctypes.c_double),
                ("local_mean", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class HeaderC(ctypes.Structure):
    _fields_ = [("fch1", ctypes.c_double), ("foff", ctypes.c_double), ("tsamp", ctypes.c_double),
                ("nchans", ctypes.c_uint32), ("_pad", ctypes.c_uint32)]


def ptr(a: np.ndarray | None) -> ctypes.c_void_p:
    """Raw pointer of a C-contiguous numpy array (or NULL)."""
    if a is None:
        return ctypes.c_void_p(0)
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)
