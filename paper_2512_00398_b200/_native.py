"""Loader and ctypes signatures of libpgb200.so (include/pulsegrid_b200.h).

The library is built in-tree (paper_2512_00398_b200/libpgb200.so, by
csrc/Makefile via __graft_entry__.build()).  There is no CPU fallback: if the
library is missing, importing this module raises, and on a machine without an
sm_100 GPU every context creation fails with DeviceError.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import abi
from .errors import raise_for

LIB_PATH = Path(__file__).resolve().parent / "libpgb200.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_2512_00398_b200/csrc).  There is no CPU fallback.")

lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)

_c = ctypes
_vp, _u32, _u64, _sz, _int = _c.c_void_p, _c.c_uint32, _c.c_uint64, _c.c_size_t, _c.c_int
_P = _c.POINTER

SIGNATURES = {
    "pgb_abi_version": ([], _int),
    "pgb_last_error": ([], _c.c_char_p),
    "pgb_device_count": ([_P(_int)], _int),
    "pgb_delay_samples": ([_c.c_double, _P(abi.HeaderC), _u32], _c.c_int64),
    "pgb_adaptive_dm_step": ([_c.c_double, _P(abi.HeaderC)], _c.c_double),
    "pgb_generate_dm_trials": ([_c.c_double, _c.c_double, _P(abi.HeaderC), _int, _c.c_double, _vp,
                                _vp, _sz, _P(_sz)], _int),
    "pgb_create": ([_int, _P(_vp)], _int),
    "pgb_destroy": ([_vp], _int),
    "pgb_set_plan": ([_vp, _vp, _vp, _u32, _u32], _int),
    "pgb_set_trial_range": ([_vp, _u32, _u32], _int),
    "pgb_run_dm_loop_u8": ([_vp, _vp, _int, _P(abi.ChunkSpecC), _P(abi.EngineConfigC), _P(_sz),
                            _P(_sz)], _int),
    "pgb_run_dm_loop_f32": ([_vp, _vp, _int, _P(abi.ChunkSpecC), _P(abi.EngineConfigC), _P(_sz),
                             _P(_sz)], _int),
    "pgb_fetch_candidates": ([_vp, _vp, _sz], _int),
    "pgb_fetch_skipped": ([_vp, _vp, _sz], _int),
    "pgb_device_candidates": ([_vp, _P(_vp), _P(_sz)], _int),
    "pgb_dedisperse_u8": ([_vp, _vp, _u64, _u32, _u32, _vp, _u64], _int),
    "pgb_dedisperse_f32": ([_vp, _vp, _u64, _u32, _u32, _vp, _u64], _int),
    "pgb_link_grid": ([_vp, _vp, _int, _sz, _P(abi.LinkRadiiC), _P(_sz)], _int),
    "pgb_fetch_clusters": ([_vp, _vp, _sz, _vp, _sz], _int),
    "pgb_search_file_u8": ([_vp, _vp, _int, _u64, _vp, _sz, _P(abi.EngineConfigC),
                            _P(abi.LinkRadiiC), _P(abi.RfiConfigC), _P(_sz), _P(_sz)], _int),
    "pgb_rfi_clean": ([_vp, _vp, _int, _int, _u64, _P(abi.RfiConfigC), _vp, _P(_u64), _P(_u64)], _int),
    "pgb_fetch_rfi_flags": ([_vp, _vp, _vp], _int),
    "pgb_fetch_file_candidates": ([_vp, _vp, _sz], _int),
    "pgb_fetch_file_skipped": ([_vp, _vp, _sz, _P(_sz)], _int),
    "pgb_launch_count": ([_vp, _P(_u64)], _int),
    "pgb_last_dedisp_time": ([_vp, _P(_c.c_double), _P(_u64), _P(_u64)], _int),
    "pgb_stream": ([_vp, _P(_vp)], _int),
    "pgb_last_cluster_ms": ([_vp, _P(_c.c_double)], _int),
    "pgb_last_stage_times": ([_vp, _P(_c.c_double)], _int),
    "pgb_microbench_add_peak": ([_int, _P(_c.c_double), _vp], _int),
    "pgb_stream_begin": ([_vp, _u64, _vp, _sz, _P(abi.EngineConfigC), _P(abi.LinkRadiiC),
                          _P(abi.RfiConfigC)], _int),
    "pgb_stream_buffer": ([_vp, _sz, _P(_vp), _P(_sz)], _int),
    "pgb_stream_push": ([_vp, _sz, _vp], _int),
    "pgb_stream_upload": ([_vp, _sz], _int),
    "pgb_stream_upload_part": ([_vp, _sz, _sz, _sz, _int], _int),
    "pgb_stream_finish": ([_vp, _P(_sz), _P(_sz)], _int),
    "pgb_device_alloc": ([_int, _sz, _P(_vp)], _int),
    "pgb_device_free": ([_int, _vp], _int),
    "pgb_ipc_get_handle": ([_vp, _vp], _int),
    "pgb_ipc_open": ([_int, _vp, _P(_vp)], _int),
    "pgb_ipc_close": ([_vp], _int),
    "pgb_copy_async": ([_vp, _vp, _vp, _sz], _int),
    "pgb_synchronize": ([_vp], _int),
}

def _bind(handle: ctypes.CDLL) -> ctypes.CDLL:
    for name, (args, res) in SIGNATURES.items():
        f = getattr(handle, name)
        f.argtypes = args
        f.restype = res
    return handle


_bind(lib)

ABLATION_LIB_PATH = LIB_PATH.with_name("libpgb200_ablations.so")
_ablation = None


def ablation_lib() -> ctypes.CDLL:
    """libpgb200_ablations.so (csrc/Makefile, -DPGB_ABLATIONS): the product path plus the
    PGB_* switchable alternatives.  Loaded only on request, never by the product path."""
    global _ablation
    if _ablation is None:
        if not ABLATION_LIB_PATH.exists():
            raise ImportError(f"{ABLATION_LIB_PATH} is not built (make -C paper_2512_00398_b200/csrc)")
        _ablation = _bind(ctypes.CDLL(str(ABLATION_LIB_PATH), mode=os.RTLD_LOCAL))
    return _ablation


def check(rc: int, handle: ctypes.CDLL | None = None) -> None:
    """Raise the pulsegrid exception named by a pgb_status (message from `handle`'s
    thread-local last error; default: the product library)."""
    if rc:
        raise_for(rc, (handle or lib).pgb_last_error().decode(errors="replace"))


def device_count() -> int:
    n = _int(0)
    check(lib.pgb_device_count(_c.byref(n)))
    return n.value


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
