"""ctypes front-end of the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two checkers with one interface:

* ``Reference`` -- the unmodified reference library compiled from
  /root/reference/proj/src (oracle/_ref/libpgref.so, built by oracle/Makefile),
  driven through its own public API by oracle/ref_harness.cpp.
* ``Port``      -- our plain-C restatement (oracle/pg_oracle.c ->
  oracle/_build/libpgoracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
import this module.  The product never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2512_00398_b200 import abi

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libpgref.so"
REF_NATIVE_SO = HERE / "_ref" / "native" / "libpgref.so"
PORT_SO = HERE / "_build" / "libpgoracle.so"

_c = ctypes
_vp = _c.c_void_p
_u64 = _c.c_uint64
_u32 = _c.c_uint32
_sz = _c.c_size_t


def build(native: bool = False) -> None:
    """Build the oracles (the restatement always; the reference only where
    /root/reference exists, i.e. in the dev container)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if Path("/root/reference/proj/src").is_dir():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
        if (HERE.parent / "paper_2512_00398_b200" / "libpgb200.so").exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "dropin"], check=True)
        if native:
            subprocess.run(["make", "-s", "-C", str(HERE), "native"], check=True)


def _header(fch1, foff, tsamp, nchans):
    return abi.HeaderC(float(fch1), float(foff), float(tsamp), int(nchans), 0)


def _spec(spec) -> abi.ChunkSpecC:
    if isinstance(spec, abi.ChunkSpecC):
        return spec
    return abi.ChunkSpecC(*(int(spec[k]) for k in
                            ("index", "start_sample", "length", "overlap", "valid_begin", "valid_end")))


def _cfg(cfg) -> abi.EngineConfigC:
    if isinstance(cfg, abi.EngineConfigC):
        return cfg
    return abi.EngineConfigC(int(cfg.get("n_workers", 1)), float(cfg.get("detect_thresh", 6.0)),
                             float(cfg.get("tsamp", 0.0)), int(cfg.get("boxcar_max", 4096)),
                             int(cfg.get("baseline_window", 0)),
                             int(cfg.get("memory_budget", 2 << 30)),
                             int(cfg.get("max_in_flight", 0)))


def _radii(r) -> abi.LinkRadiiC:
    if r is None:
        r = (3, 9, 3)
    if isinstance(r, dict):
        r = (r["sep_time"], r["sep_dm_trials"], r["sep_width"])
    return abi.LinkRadiiC(int(r[0]), int(r[1]), int(r[2]))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Base:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run oracle.pyoracle.build())")
        self.lib = ctypes.CDLL(str(path))
        self.path = path
        self._free = getattr(self.lib, self.prefix + "free")
        self._free.argtypes = [_vp]

    def _fn(self, name, argtypes, restype=_c.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._errmsg())

    def _errmsg(self) -> str:
        return ""

    def _take(self, p: _vp, n: int, dtype) -> np.ndarray:
        if n:
            buf = (ctypes.c_char * (n * np.dtype(dtype).itemsize)).from_address(p.value)
            out = np.frombuffer(bytes(buf), dtype=dtype).copy()
        else:
            out = np.zeros(0, dtype=dtype)
        if p.value:
            self._free(p)
        return out

    # ---- plan -------------------------------------------------------------
    def delay_samples(self, dm, fch1, foff, tsamp, nchans, channel) -> int:
        f = self._fn("delay_samples", [_c.c_double, _c.POINTER(abi.HeaderC), _u32], _c.c_int64)
        h = _header(fch1, foff, tsamp, nchans)
        return int(f(dm, _c.byref(h), channel))

    def adaptive_dm_step(self, tol, fch1, foff, tsamp, nchans) -> float:
        f = self._fn("adaptive_dm_step", [_c.c_double, _c.POINTER(abi.HeaderC)], _c.c_double)
        h = _header(fch1, foff, tsamp, nchans)
        return float(f(tol, _c.byref(h)))

    def generate_dm_trials(self, dm_lo, dm_hi, fch1, foff, tsamp, nchans, *, step=None, tol=None):
        f = self._fn("generate_dm_trials", [_c.c_double, _c.c_double, _c.POINTER(abi.HeaderC),
                                            _c.c_int, _c.c_double, _vp, _vp, _sz, _c.POINTER(_sz)])
        h = _header(fch1, foff, tsamp, nchans)
        kind, val = (abi.SPACING_LINEAR, step) if step is not None else (abi.SPACING_ADAPTIVE, tol)
        n = _sz(0)
        self._check(f(dm_lo, dm_hi, _c.byref(h), kind, val, None, None, 0, _c.byref(n)))
        dms = np.zeros(n.value, np.float64)
        delays = np.zeros((n.value, nchans), np.int64)
        self._check(f(dm_lo, dm_hi, _c.byref(h), kind, val, abi.ptr(dms), abi.ptr(delays), n.value,
                      _c.byref(n)))
        return dms, delays

    def plan_chunks(self, nsamples, chunk_len, overlap) -> np.ndarray:
        f = self._fn("plan_chunks", [_u64, _u64, _u64, _vp, _sz, _c.POINTER(_sz)])
        n = _sz(0)
        self._check(f(nsamples, chunk_len, overlap, None, 0, _c.byref(n)))
        out = np.zeros(n.value, abi.CHUNK_SPEC_DTYPE)
        self._check(f(nsamples, chunk_len, overlap, abi.ptr(out), n.value, _c.byref(n)))
        return out


class Reference(_Base):
    """The compiled reference library (oracle/_ref)."""

    prefix = "pgref_"

    def __init__(self, native: bool = False):
        super().__init__(REF_NATIVE_SO if native else REF_SO)
        self.lib.pgref_last_error.restype = _c.c_char_p

    def _errmsg(self):
        return self.lib.pgref_last_error().decode()

    def run_dm_loop(self, data: np.ndarray, spec, dms, delays, cfg, *, parity=True):
        """Returns (candidates, skipped, wall_ms)."""
        data = np.ascontiguousarray(data)
        kind = "u8" if data.dtype == np.uint8 else "f32"
        if kind == "f32":
            data = np.ascontiguousarray(data, dtype=np.float32)
        f = self._fn("run_dm_loop_" + kind,
                     [_vp, _c.POINTER(abi.ChunkSpecC), _u32, _vp, _vp, _u32,
                      _c.POINTER(abi.EngineConfigC), _c.c_int, _c.POINTER(_vp), _c.POINTER(_sz),
                      _c.POINTER(_vp), _c.POINTER(_sz), _c.POINTER(_c.c_double)])
        dms = np.ascontiguousarray(dms, np.float64)
        delays = np.ascontiguousarray(delays, np.int64)
        sp, cf = _spec(spec), _cfg(cfg)
        pc, nc, ps, ns, ms = _vp(), _sz(), _vp(), _sz(), _c.c_double()
        self._check(f(abi.ptr(data), _c.byref(sp), delays.shape[1], abi.ptr(dms), abi.ptr(delays),
                      delays.shape[0], _c.byref(cf), int(parity), _c.byref(pc), _c.byref(nc),
                      _c.byref(ps), _c.byref(ns), _c.byref(ms)))
        return (self._take(pc, nc.value, abi.CANDIDATE_DTYPE), self._take(ps, ns.value, np.uint64),
                ms.value)

    def dedisperse(self, data: np.ndarray, dms, delays, trial: int) -> np.ndarray:
        data = np.ascontiguousarray(data, np.float32)
        L, nch = data.shape
        f = self._fn("dedisperse", [_vp, _u64, _u32, _vp, _vp, _u32, _u32, _vp, _c.POINTER(_u64)])
        delays = np.ascontiguousarray(delays, np.int64)
        out = np.zeros(L, np.float32)
        n = _u64()
        self._check(f(abi.ptr(data), L, nch, abi.ptr(np.ascontiguousarray(dms, np.float64)),
                      abi.ptr(delays), delays.shape[0], trial, abi.ptr(out), _c.byref(n)))
        return out[: n.value]

    def dedisperse_block(self, data: np.ndarray, dms, delays, trials) -> list[np.ndarray]:
        data = np.ascontiguousarray(data, np.float32)
        L, nch = data.shape
        f = self._fn("dedisperse_block", [_vp, _u64, _u32, _vp, _vp, _u32, _vp, _u32, _vp, _u64])
        delays = np.ascontiguousarray(delays, np.int64)
        tr = np.ascontiguousarray(trials, np.uint64)
        out = np.zeros((len(tr), L), np.float32)
        self._check(f(abi.ptr(data), L, nch, abi.ptr(np.ascontiguousarray(dms, np.float64)),
                      abi.ptr(delays), delays.shape[0], abi.ptr(tr), len(tr), abi.ptr(out), L))
        return [out[b, : L - int(delays[t].max())] for b, t in enumerate(tr)]

    def remove_baseline(self, x: np.ndarray, window: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        f = self._fn("remove_baseline", [_vp, _u64, _u64, _vp])
        self._check(f(abi.ptr(x), len(x), window, abi.ptr(out)))
        return out

    def normalize_to_sums(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float32)
        n = len(x)
        sums = np.zeros(n, np.float64)
        maxima = np.zeros((n + 63) // 64 + 1, np.float64)
        rms = _c.c_double()
        f = self._fn("normalize_to_sums", [_vp, _u64, _vp, _vp, _c.POINTER(_c.c_double)])
        self._check(f(abi.ptr(x), n, abi.ptr(sums), abi.ptr(maxima), _c.byref(rms)))
        return sums, rms.value

    def find_peaks(self, snr: np.ndarray, threshold: float, width_index: int, *, start_sample=0,
                   tsamp=64e-6, dm_trial=0, dm=0.0, valid_begin=0, valid_end=None,
                   drop_left=False, drop_right=False) -> np.ndarray:
        snr = np.ascontiguousarray(snr, np.float64)
        if valid_end is None:
            valid_end = start_sample + len(snr)
        f = self._fn("find_peaks", [_vp, _u64, _c.c_double, _u32, _u64, _c.c_double, _u32,
                                    _c.c_double, _u64, _u64, _c.c_int, _c.c_int, _c.POINTER(_vp),
                                    _c.POINTER(_sz)])
        pc, nc = _vp(), _sz()
        self._check(f(abi.ptr(snr), len(snr), threshold, width_index, start_sample, tsamp, dm_trial,
                      dm, valid_begin, valid_end, int(drop_left), int(drop_right), _c.byref(pc),
                      _c.byref(nc)))
        return self._take(pc, nc.value, abi.CANDIDATE_DTYPE)

    def link_grid(self, cands: np.ndarray, radii=None, *, reference=False):
        """Returns (clusters, member_ids, wall_ms)."""
        cands = np.ascontiguousarray(cands, abi.CANDIDATE_DTYPE)
        f = self._fn("link_grid", [_vp, _sz, _c.POINTER(abi.LinkRadiiC), _c.c_int, _c.POINTER(_vp),
                                   _c.POINTER(_sz), _c.POINTER(_vp), _c.POINTER(_c.c_double)])
        r = _radii(radii)
        pc, nc, pm, ms = _vp(), _sz(), _vp(), _c.c_double()
        self._check(f(abi.ptr(cands), len(cands), _c.byref(r), int(reference), _c.byref(pc),
                      _c.byref(nc), _c.byref(pm), _c.byref(ms)))
        clusters = self._take(pc, nc.value, abi.CLUSTER_DTYPE)
        nm = int(clusters["members"].sum()) if len(clusters) else 0
        return clusters, self._take(pm, nm, np.uint64), ms.value

    def write_candidates(self, clusters: np.ndarray) -> str:
        clusters = np.ascontiguousarray(clusters, abi.CLUSTER_DTYPE)
        f = self._fn("write_candidates", [_vp, _sz, _c.POINTER(_c.c_char_p), _c.POINTER(_sz)])
        txt, n = _c.c_char_p(), _sz()
        self._check(f(abi.ptr(clusters), len(clusters), _c.byref(txt), _c.byref(n)))
        s = txt.value.decode() if n.value else ""
        self._free(_c.cast(txt, _vp))
        return s

    def generate_noise(self, fch1, foff, tsamp, nchans, nsamples, mean, sigma, seed) -> np.ndarray:
        out = np.zeros((nsamples, nchans), np.float32)
        f = self._fn("generate_noise", [_c.POINTER(abi.HeaderC), _u64, _c.c_float, _c.c_float,
                                        _u64, _vp])
        h = _header(fch1, foff, tsamp, nchans)
        self._check(f(_c.byref(h), nsamples, mean, sigma, seed, abi.ptr(out)))
        return out

    def inject_pulse(self, grid: np.ndarray, fch1, foff, tsamp, dm, t0, width, amplitude):
        assert grid.dtype == np.float32 and grid.flags["C_CONTIGUOUS"]
        f = self._fn("inject_pulse", [_vp, _u64, _c.POINTER(abi.HeaderC), _c.c_double, _c.c_double,
                                      _u64, _c.c_float])
        h = _header(fch1, foff, tsamp, grid.shape[1])
        self._check(f(abi.ptr(grid), grid.shape[0], _c.byref(h), dm, t0, width, amplitude))

    def rfi(self, data: np.ndarray, *, narrowband=True, broadband=True, k_sigma=6.0, k_mad=5.0,
            local_mean=True):
        """(cleaned float chunk, bad-channel mask, bad-sample mask) of the reference RFI stage."""
        x = np.ascontiguousarray(data, np.float32).copy()
        L, nch = x.shape
        bc = np.zeros(nch, np.uint8)
        bs = np.zeros(L, np.uint8)
        f = self._fn("rfi", [_vp, _u64, _u32, _c.c_int, _c.c_int, _c.c_double, _c.c_double, _c.c_int,
                             _vp, _vp])
        self._check(f(abi.ptr(x), L, nch, int(narrowband), int(broadband), k_sigma, k_mad,
                      int(local_mean), abi.ptr(bc), abi.ptr(bs)))
        return x, bc.astype(bool), bs.astype(bool)

    def amplitude_for_snr(self, snr, sigma, nchans, width) -> float:
        f = self._fn("amplitude_for_snr", [_c.c_double, _c.c_double, _u32, _u64], _c.c_double)
        return float(f(snr, sigma, nchans, width))

    def write_filterbank(self, path, grid: np.ndarray, fch1, foff, tsamp, nbits=8):
        grid = np.ascontiguousarray(grid, np.float32)
        f = self._fn("write_filterbank", [_c.c_char_p, _c.POINTER(abi.HeaderC), _u32, _vp, _u64])
        h = _header(fch1, foff, tsamp, grid.shape[1])
        self._check(f(str(path).encode(), _c.byref(h), nbits, abi.ptr(grid), grid.shape[0]))

    class SearchParams(ctypes.Structure):
        _fields_ = [("dm_lo", _c.c_double), ("dm_hi", _c.c_double), ("dm_step", _c.c_double),
                    ("n_workers", _u32), ("detect_thresh", _c.c_float), ("boxcar_max", _u64),
                    ("baseline_len_s", _c.c_double), ("nsamps_chunk", _u64),
                    ("rfi_narrowband", _c.c_int), ("rfi_broadband", _c.c_int),
                    ("k_sigma", _c.c_double), ("k_mad", _c.c_double), ("parity", _c.c_int),
                    ("radii", abi.LinkRadiiC)]

    def _params(self, **kw):
        p = self.SearchParams()
        p.dm_lo = kw.get("dm_lo", 0.0)
        p.dm_hi = kw.get("dm_hi", 1000.0)
        p.dm_step = kw["dm_step"]
        p.n_workers = kw.get("n_workers", os.cpu_count() or 1)
        p.detect_thresh = kw.get("detect_thresh", 6.0)
        p.boxcar_max = kw.get("boxcar_max", 4096)
        p.baseline_len_s = kw.get("baseline_len_s", 2.0)
        p.nsamps_chunk = kw.get("nsamps_chunk", 1 << 18)
        p.rfi_narrowband = int(kw.get("rfi_narrowband", False))
        p.rfi_broadband = int(kw.get("rfi_broadband", False))
        p.k_sigma = kw.get("k_sigma", 6.0)
        p.k_mad = kw.get("k_mad", 5.0)
        p.parity = int(kw.get("parity", True))
        p.radii = _radii(kw.get("radii"))
        return p

    def execute_file(self, path, out_path, **kw):
        """create_task + execute_task; returns (n_clusters, stage_ms dict)."""
        f = self._fn("execute_file", [_c.c_char_p, _c.c_char_p, _c.POINTER(self.SearchParams), _vp,
                                      _c.POINTER(_sz)])
        p = self._params(**kw)
        ms = np.zeros(6, np.float64)
        n = _sz()
        self._check(f(str(path).encode(), str(out_path).encode(), _c.byref(p), abi.ptr(ms),
                      _c.byref(n)))
        keys = ("wall", "read", "rfi", "dm_loop", "cluster", "write")
        return n.value, dict(zip(keys, ms.tolist()))

    def search_file(self, path, **kw):
        """execute_task's body on a file with structured results (parity mode by default).

        Returns dict(candidates, clusters, members, skipped [k,2], cand_text, stage_ms)."""
        f = self._fn("search_file", [_c.c_char_p, _c.POINTER(self.SearchParams), _c.POINTER(_vp),
                                     _c.POINTER(_sz), _c.POINTER(_vp), _c.POINTER(_sz),
                                     _c.POINTER(_vp), _c.POINTER(_vp), _c.POINTER(_sz),
                                     _c.POINTER(_vp), _c.POINTER(_sz), _vp])
        p = self._params(**kw)
        pc, nc, pcl, ncl, pm, ps, ns, pt, nt = _vp(), _sz(), _vp(), _sz(), _vp(), _vp(), _sz(), _vp(), _sz()
        ms = np.zeros(4, np.float64)
        self._check(f(str(path).encode(), _c.byref(p), _c.byref(pc), _c.byref(nc), _c.byref(pcl),
                      _c.byref(ncl), _c.byref(pm), _c.byref(ps), _c.byref(ns), _c.byref(pt),
                      _c.byref(nt), abi.ptr(ms)))
        cands = self._take(pc, nc.value, abi.CANDIDATE_DTYPE)
        clusters = self._take(pcl, ncl.value, abi.CLUSTER_DTYPE)
        members = self._take(pm, int(clusters["members"].sum()) if len(clusters) else 0, np.uint64)
        skipped = self._take(ps, 2 * ns.value, np.uint64).reshape(-1, 2)
        text = self._take(pt, nt.value, np.uint8).tobytes().decode()
        return dict(candidates=cands, clusters=clusters, members=members, skipped=skipped,
                    cand_text=text, stage_ms=dict(zip(("read", "rfi", "dm_loop", "cluster"), ms.tolist())))

    def create_task_plan(self, path, **kw):
        """(chunk specs, baseline_window) create_task resolves for a file."""
        f = self._fn("create_task_plan", [_c.c_char_p, _c.POINTER(self.SearchParams), _vp, _sz,
                                          _c.POINTER(_sz), _c.POINTER(_u64)])
        p = self._params(**kw)
        n, bw = _sz(), _u64()
        self._check(f(str(path).encode(), _c.byref(p), None, 0, _c.byref(n), _c.byref(bw)))
        out = np.zeros(n.value, abi.CHUNK_SPEC_DTYPE)
        self._check(f(str(path).encode(), _c.byref(p), abi.ptr(out), n.value, _c.byref(n),
                      _c.byref(bw)))
        return out, int(bw.value)


class Port(_Base):
    """The plain-C restatement (oracle/pg_oracle.c)."""

    prefix = "pgo_"

    def __init__(self):
        super().__init__(PORT_SO)

    def run_dm_loop(self, data: np.ndarray, spec, dms, delays, cfg):
        data = np.ascontiguousarray(data)
        kind = "u8" if data.dtype == np.uint8 else "f32"
        if kind == "f32":
            data = np.ascontiguousarray(data, dtype=np.float32)
        f = self._fn("run_dm_loop_" + kind,
                     [_vp, _c.POINTER(abi.ChunkSpecC), _u32, _vp, _vp, _u32,
                      _c.POINTER(abi.EngineConfigC), _c.POINTER(_vp), _c.POINTER(_sz),
                      _c.POINTER(_vp), _c.POINTER(_sz)])
        dms = np.ascontiguousarray(dms, np.float64)
        delays = np.ascontiguousarray(delays, np.int64)
        sp, cf = _spec(spec), _cfg(cfg)
        pc, nc, ps, ns = _vp(), _sz(), _vp(), _sz()
        self._check(f(abi.ptr(data), _c.byref(sp), delays.shape[1], abi.ptr(dms), abi.ptr(delays),
                      delays.shape[0], _c.byref(cf), _c.byref(pc), _c.byref(nc), _c.byref(ps),
                      _c.byref(ns)))
        return self._take(pc, nc.value, abi.CANDIDATE_DTYPE), self._take(ps, ns.value, np.uint64)

    def dedisperse(self, data: np.ndarray, delays_row: np.ndarray) -> np.ndarray:
        data = np.ascontiguousarray(data, np.float32)
        L, nch = data.shape
        d = np.ascontiguousarray(delays_row, np.int64)
        out = np.zeros(L, np.float32)
        f = self._fn("dedisperse", [_vp, _u64, _u32, _vp, _vp], None)
        f(abi.ptr(data), L, nch, abi.ptr(d), abi.ptr(out))
        return out[: L - int(d.max())]

    def remove_baseline(self, x: np.ndarray, window: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        f = self._fn("remove_baseline", [_vp, _u64, _u64, _vp], None)
        f(abi.ptr(x), len(x), window, abi.ptr(out))
        return out

    def normalize_to_sums(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float32)
        sums = np.zeros(len(x), np.float64)
        rms = _c.c_double()
        f = self._fn("normalize_to_sums", [_vp, _u64, _vp, _c.POINTER(_c.c_double)])
        self._check(f(abi.ptr(x), len(x), abi.ptr(sums), _c.byref(rms)))
        return sums, rms.value

    def link_grid(self, cands: np.ndarray, radii=None):
        cands = np.ascontiguousarray(cands, abi.CANDIDATE_DTYPE)
        f = self._fn("link_grid", [_vp, _sz, _c.POINTER(abi.LinkRadiiC), _c.POINTER(_vp),
                                   _c.POINTER(_sz), _c.POINTER(_vp)])
        r = _radii(radii)
        pc, nc, pm = _vp(), _sz(), _vp()
        self._check(f(abi.ptr(cands), len(cands), _c.byref(r), _c.byref(pc), _c.byref(nc),
                      _c.byref(pm)))
        clusters = self._take(pc, nc.value, abi.CLUSTER_DTYPE)
        return clusters, self._take(pm, len(cands), np.uint64)

    def format_candidates(self, clusters: np.ndarray) -> str:
        clusters = np.ascontiguousarray(clusters, abi.CLUSTER_DTYPE)
        f = self._fn("format_candidates", [_vp, _sz, _vp, _sz], _sz)
        n = f(abi.ptr(clusters), len(clusters), None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        f(abi.ptr(clusters), len(clusters), buf, n + 1)
        return buf.value.decode()
