"""The DM loop: pulsegrid's engine.hpp API on the B200.

`run_dm_loop(chunk, plan, cfg)` is the drop-in for
pulsegrid::run_dm_loop (/root/reference/proj/include/pulsegrid/engine.hpp:61-62,
src/engine.cpp:85-265): same inputs (a time-major chunk with its ChunkSpec, the
DM plan, the engine config), same output (candidates sorted by
(peak_sample, dm_trial, width_index) plus the sorted skipped trials), same
exceptions.  The work runs in libpgb200 on one CUDA device; there is no CPU path.

Differences that are deliberate and documented in DESIGN.md:
* n_workers / memory_budget / max_in_flight are validated like the reference but
  do not change how the device batches trials (results never depended on them);
* the BufferPool argument is accepted and ignored: device memory comes from the
  engine's own arena.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import abi
from ._native import ablation_lib, check, lib
from .dedisp import DmTrialPlan


@dataclass
class ChunkSpec:
    """pulsegrid::ChunkSpec (filterbank.hpp:48-55)."""

    index: int = 0
    start_sample: int = 0
    length: int = 0
    overlap: int = 0
    valid_begin: int = 0
    valid_end: int = 0

    def _c(self) -> abi.ChunkSpecC:
        return abi.ChunkSpecC(self.index, self.start_sample, self.length, self.overlap,
                              self.valid_begin, self.valid_end)

    @staticmethod
    def whole(length: int, start: int = 0) -> "ChunkSpec":
        """The spec tests/oracles.hpp:make_chunk builds (valid range = the chunk)."""
        return ChunkSpec(0, start, length, 0, start, start + length)


@dataclass
class Chunk:
    """pulsegrid::Chunk (filterbank.hpp:59-67): time-major [length][nchans] samples.

    `data` may be uint8 codes (the raw 8-bit payload -- exact integer path), float32
    (widened samples; exact in-order fp32 path), or a CUDA torch tensor of either
    dtype already resident on the engine's device.
    """

    spec: ChunkSpec
    data: object

    @property
    def nchans(self) -> int:
        return int(self.data.shape[1])


@dataclass
class LinkRadii:
    """pulsegrid::LinkRadii (cluster.hpp:13-17)."""

    sep_time: int = 3
    sep_dm_trials: int = 9
    sep_width: int = 3

    def _c(self) -> abi.LinkRadiiC:
        return abi.LinkRadiiC(self.sep_time, self.sep_dm_trials, self.sep_width)


@dataclass
class RfiConfig:
    """The RFI fields of pulsegrid::SearchParams (pipeline.hpp:31-35); reference defaults."""

    narrowband: bool = True
    broadband: bool = True
    k_sigma: float = 6.0
    k_mad: float = 5.0
    local_mean: bool = True  # MaskPolicy::local_mean (False = zero)

    def _c(self) -> abi.RfiConfigC:
        return abi.RfiConfigC(int(self.narrowband), int(self.broadband), float(self.k_sigma),
                              float(self.k_mad), int(self.local_mean), 0)

    @property
    def active(self) -> bool:
        return bool(self.narrowband or self.broadband)


@dataclass
class TrialTiming:
    """pulsegrid::TrialTiming (engine.hpp:16-23); device stages are amortized per trial."""

    trial: int = 0
    dedisperse_ms: float = 0.0
    baseline_ms: float = 0.0
    normalize_ms: float = 0.0
    boxcar_ms: float = 0.0
    peaks_ms: float = 0.0


@dataclass
class EngineConfig:
    """pulsegrid::EngineConfig (engine.hpp:25-35)."""

    n_workers: int = 1
    tsamp: float = 0.0
    detect_thresh: float = 6.0
    boxcar_max: int = 4096
    baseline_window: int = 0
    radii: LinkRadii = field(default_factory=LinkRadii)
    memory_budget: int = 2 << 30
    max_in_flight: int = 0
    timing_sink: Callable[[TrialTiming], None] | None = None

    def _c(self) -> abi.EngineConfigC:
        return abi.EngineConfigC(int(self.n_workers), float(self.detect_thresh), float(self.tsamp),
                                 int(self.boxcar_max), int(self.baseline_window),
                                 int(self.memory_budget), int(self.max_in_flight))


@dataclass
class DmLoopResult:
    """pulsegrid::DmLoopResult (engine.hpp:37-40), as numpy arrays."""

    candidates: np.ndarray       # abi.CANDIDATE_DTYPE, sorted by (peak, trial, width)
    skipped_trials: np.ndarray   # uint64, ascending


def partition_trials(ntrials: int, n_workers: int) -> list[list[int]]:
    """src/engine.cpp:53-58 (kept for API parity; the device does not partition)."""
    parts: list[list[int]] = [[] for _ in range(max(1, n_workers))]
    for i in range(ntrials):
        parts[i % len(parts)].append(i)
    return parts


def _aligned(n: int) -> int:
    v = max(n, 256)
    return 1 << (v - 1).bit_length()


def trial_working_set_bytes(plan: DmTrialPlan, chunk_len: int, cfg: EngineConfig) -> int:
    """src/engine.cpp:60-73."""
    min_delay = plan.trial_max_delay(0)
    longest = chunk_len - min_delay if chunk_len > min_delay else 1
    series = _aligned(longest * 4)
    n_blocks = (longest + 63) // 64
    sums = _aligned((longest + n_blocks) * 8)
    return (2 if cfg.baseline_window > 0 else 1) * series + sums


def in_flight_limit(plan: DmTrialPlan, chunk_len: int, cfg: EngineConfig) -> int:
    """src/engine.cpp:75-83."""
    from .errors import ConfigError

    ws = trial_working_set_bytes(plan, chunk_len, cfg)
    limit = cfg.memory_budget // ws
    if limit == 0:
        raise ConfigError(f"memory budget of {cfg.memory_budget} bytes is below one trial's "
                          f"working set ({ws})")
    return limit


class DeviceBuffer:
    """A dedicated device allocation (pgb_device_alloc) holding a [rows][nchans] u8 payload.

    Usable as a `search_file` payload like a CUDA tensor, and exportable to the other
    ranks of a node over CUDA IPC (its handle maps exactly this buffer)."""

    def __init__(self, device: int, shape: tuple[int, int]):
        self.device = int(device)
        self.shape = (int(shape[0]), int(shape[1]))
        self.nbytes = self.shape[0] * self.shape[1]
        p = ctypes.c_void_p()
        check(lib.pgb_device_alloc(self.device, self.nbytes, ctypes.byref(p)))
        self.ptr = int(p.value)

    def ipc_handle(self) -> bytes:
        h = (ctypes.c_uint8 * 64)()
        check(lib.pgb_ipc_get_handle(ctypes.c_void_p(self.ptr), h))
        return bytes(h)

    def free(self) -> None:
        if self.ptr:
            check(lib.pgb_device_free(self.device, ctypes.c_void_p(self.ptr)))
            self.ptr = 0


def _device_tensor(x):
    """(data_ptr, is_u8, device) for a CUDA torch tensor or a DeviceBuffer, else None."""
    if isinstance(x, DeviceBuffer):
        return x.ptr, True, x.device
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return None
        if not x.is_contiguous():
            raise ValueError("device chunk must be contiguous")
        if x.dtype not in (torch.uint8, torch.float32):
            raise TypeError("device chunk must be uint8 or float32")
        return x.data_ptr(), x.dtype == torch.uint8, x.device.index or 0
    return None


class Engine:
    """One libpgb200 context: a CUDA stream plus a device arena on one GPU."""

    def __init__(self, device: int = 0, *, ablations: bool = False):
        """ablations=True binds libpgb200_ablations.so instead of the product library: the
        same path plus the alternative kernels and schedules of DESIGN.md section 10,
        selected by PGB_* environment switches (tests and tools only)."""
        self.device = device
        self._lib = ablation_lib() if ablations else lib
        h = ctypes.c_void_p()
        self._check(self._lib.pgb_create(int(device), ctypes.byref(h)))
        self._h = h
        self._plan_key = None
        self._range = None

    def _check(self, rc: int) -> None:
        check(rc, self._lib)

    # ---- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if self._h:
            self._lib.pgb_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- plan ------------------------------------------------------------------
    def set_plan(self, plan: DmTrialPlan, trial_range: tuple[int, int] | None = None) -> None:
        key = (id(plan), plan.ntrials, plan.nchans, plan.delays.ctypes.data)
        if key != self._plan_key:
            self._check(self._lib.pgb_set_plan(self._h, abi.ptr(plan.dms), abi.ptr(plan.delays),
                                   plan.ntrials, plan.nchans))
            self._plan_key = key
            self._plan_ref = plan  # keep the arrays alive while the key is cached
            self._range = None
        rng = trial_range if trial_range is not None else (0, plan.ntrials)
        if rng != self._range:
            self._check(self._lib.pgb_set_trial_range(self._h, int(rng[0]), int(rng[1])))
            self._range = rng

    # ---- run_dm_loop -------------------------------------------------------------
    def run_dm_loop(self, chunk: Chunk, plan: DmTrialPlan, cfg: EngineConfig,
                    pool=None, *, trial_range: tuple[int, int] | None = None) -> DmLoopResult:
        del pool  # device arena replaces the host BufferPool
        self.set_plan(plan, trial_range)
        spec = chunk.spec._c()
        ccfg = cfg._c()
        nc, ns = ctypes.c_size_t(), ctypes.c_size_t()
        dev = _device_tensor(chunk.data)
        if dev is not None:
            ptr, is_u8, _ = dev
            import torch

            torch.cuda.current_stream().synchronize()
            fn = self._lib.pgb_run_dm_loop_u8 if is_u8 else self._lib.pgb_run_dm_loop_f32
            check(fn(self._h, ctypes.c_void_p(ptr), 1, ctypes.byref(spec), ctypes.byref(ccfg),
                     ctypes.byref(nc), ctypes.byref(ns)))
        else:
            data = np.asarray(chunk.data)
            if data.ndim != 2 or data.shape[1] != plan.nchans:
                raise ValueError("chunk data must be [length][nchans] matching the plan")
            if data.shape[0] < chunk.spec.length:
                raise ValueError("chunk data shorter than spec.length")
            if data.dtype == np.uint8:
                data = np.ascontiguousarray(data)
                fn = self._lib.pgb_run_dm_loop_u8
            else:
                data = np.ascontiguousarray(data, dtype=np.float32)
                fn = self._lib.pgb_run_dm_loop_f32
            check(fn(self._h, abi.ptr(data), 0, ctypes.byref(spec), ctypes.byref(ccfg),
                     ctypes.byref(nc), ctypes.byref(ns)))
        cands = np.zeros(nc.value, abi.CANDIDATE_DTYPE)
        self._check(self._lib.pgb_fetch_candidates(self._h, abi.ptr(cands), nc.value))
        skipped = np.zeros(ns.value, np.uint64)
        self._check(self._lib.pgb_fetch_skipped(self._h, abi.ptr(skipped), ns.value))
        if cfg.timing_sink is not None:
            # stage times batched over the chunk, amortised over the trials that finished
            # the chain; skipped trials emit nothing (src/engine.cpp:112-118, 147-213)
            ms = (ctypes.c_double * 5)()
            self._check(self._lib.pgb_last_stage_times(self._h, ms))
            lo, hi = self._range
            done = np.setdiff1d(np.arange(lo, hi, dtype=np.uint64), skipped)
            inv = 1.0 / max(1, len(done))
            for t in done:
                cfg.timing_sink(TrialTiming(trial=int(t), dedisperse_ms=ms[0] * inv,
                                            baseline_ms=ms[1] * inv if cfg.baseline_window > 0 else 0.0,
                                            normalize_ms=ms[2] * inv, boxcar_ms=ms[3] * inv,
                                            peaks_ms=ms[4] * inv))
        return DmLoopResult(cands, skipped)

    # ---- dedispersion only --------------------------------------------------------
    def dedisperse(self, chunk_data: np.ndarray, plan: DmTrialPlan, trials: range | None = None
                   ) -> list[np.ndarray]:
        """Dedispersed series of trials [b, e) (dedisperse/dedisperse_block semantics)."""
        self.set_plan(plan)
        data = np.asarray(chunk_data)
        L = data.shape[0]
        b, e = (0, plan.ntrials) if trials is None else (trials.start, trials.stop)
        out = np.zeros((max(0, e - b), L), np.float32)
        if data.dtype == np.uint8:
            data = np.ascontiguousarray(data)
            fn = self._lib.pgb_dedisperse_u8
        else:
            data = np.ascontiguousarray(data, dtype=np.float32)
            fn = self._lib.pgb_dedisperse_f32
        check(fn(self._h, abi.ptr(data), L, b, e, abi.ptr(out), L))
        return [out[r, : L - plan.trial_max_delay(b + r)] for r in range(e - b)]

    # ---- link_grid ----------------------------------------------------------------
    def link_grid(self, cands, radii: LinkRadii | None = None) -> "Clusters":
        from .cluster import Clusters

        radii = radii or LinkRadii()
        r = radii._c()
        n = ctypes.c_size_t()
        dev = _device_tensor(cands) if not isinstance(cands, np.ndarray) else None
        if dev is not None:
            raise TypeError("pass device candidates through Engine.link_device()")
        arr = np.ascontiguousarray(cands, abi.CANDIDATE_DTYPE)
        self._check(self._lib.pgb_link_grid(self._h, abi.ptr(arr), 0, len(arr), ctypes.byref(r), ctypes.byref(n)))
        return self._fetch_clusters(n.value, len(arr))

    def link_last(self, radii: LinkRadii | None = None) -> "Clusters":
        """link_grid on the last run's device-resident candidates (no round trip)."""
        radii = radii or LinkRadii()
        r = radii._c()
        p, cnt, n = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_size_t()
        self._check(self._lib.pgb_device_candidates(self._h, ctypes.byref(p), ctypes.byref(cnt)))
        self._check(self._lib.pgb_link_grid(self._h, p, 1, cnt.value, ctypes.byref(r), ctypes.byref(n)))
        return self._fetch_clusters(n.value, cnt.value)

    def _fetch_clusters(self, ncl: int, nmem: int) -> "Clusters":
        from .cluster import Clusters

        recs = np.zeros(ncl, abi.CLUSTER_DTYPE)
        members = np.zeros(nmem, np.uint64)
        self._check(self._lib.pgb_fetch_clusters(self._h, abi.ptr(recs), ncl, abi.ptr(members), nmem))
        return Clusters(recs, members)

    # ---- file-level search ------------------------------------------------------------
    def search_file(self, payload, nsamples: int, chunks: list[ChunkSpec], plan: DmTrialPlan,
                    cfg: EngineConfig, *, trial_range: tuple[int, int] | None = None,
                    cluster: bool = True, rfi: RfiConfig | None = None):
        """execute_task's chunk loop + sort + link_grid on a raw 8-bit payload.

        Returns (candidates, clusters, skipped (chunk, trial) pairs).  cluster=False
        stops after the sorted candidates (multi-GPU shards cluster after the gather)."""
        self.set_plan(plan, trial_range)
        arr = np.zeros(len(chunks), abi.CHUNK_SPEC_DTYPE)
        for k, c in enumerate(chunks):
            arr[k] = (c.index, c.start_sample, c.length, c.overlap, c.valid_begin, c.valid_end)
        ccfg = cfg._c()
        r = cfg.radii._c()
        rp = ctypes.byref(r) if cluster else None
        nc, ncl = ctypes.c_size_t(), ctypes.c_size_t()
        dev = _device_tensor(payload)
        if dev is not None:
            if not isinstance(payload, DeviceBuffer):
                import torch

                torch.cuda.current_stream().synchronize()
            ptr, on_dev = ctypes.c_void_p(dev[0]), 1
        else:
            payload = np.ascontiguousarray(payload, dtype=np.uint8)
            ptr, on_dev = abi.ptr(payload), 0
        shape = tuple(payload.shape)
        if len(shape) != 2 or shape[1] != plan.nchans or shape[0] < nsamples:
            raise ValueError(f"payload of shape {shape} does not hold {nsamples} x {plan.nchans} samples")
        rc = rfi._c() if (rfi is not None and rfi.active) else None
        self._check(self._lib.pgb_search_file_u8(self._h, ptr, on_dev, int(nsamples), abi.ptr(arr), len(arr),
                                     ctypes.byref(ccfg), rp, ctypes.byref(rc) if rc is not None else None,
                                     ctypes.byref(nc), ctypes.byref(ncl)))
        return self.fetch_file_results(nc.value, ncl.value)

    def search_stream(self, fd: int, data_offset: int, nsamples: int, chunks: list[ChunkSpec],
                      plan: DmTrialPlan, cfg: EngineConfig, *, trial_range: tuple[int, int] | None = None,
                      cluster: bool = True, rfi: RfiConfig | None = None, read_threads: int = 8):
        """execute_task with the prefetching reader on an open 8-bit filterbank (bounded memory).

        Chunk k is read from `fd` (payload at `data_offset`, [nsamples][nchans] bytes) by
        `read_threads` parallel preads straight into the context's pinned buffer while
        chunk k-1 is pushed; host and device memory stay at two chunks
        (src/pipeline.cpp:66-106, src/filterbank.cpp:326-419)."""
        import os
        from concurrent.futures import ThreadPoolExecutor

        self.set_plan(plan, trial_range)
        arr = np.zeros(len(chunks), abi.CHUNK_SPEC_DTYPE)
        for k, c in enumerate(chunks):
            arr[k] = (c.index, c.start_sample, c.length, c.overlap, c.valid_begin, c.valid_end)
        ccfg = cfg._c()
        r = cfg.radii._c()
        rc = rfi._c() if (rfi is not None and rfi.active) else None
        self._check(self._lib.pgb_stream_begin(self._h, int(nsamples), abi.ptr(arr), len(arr), ctypes.byref(ccfg),
                                   ctypes.byref(r) if cluster else None,
                                   ctypes.byref(rc) if rc is not None else None))
        C = plan.nchans
        pool = ThreadPoolExecutor(max(1, read_threads))

        def fill(k: int) -> None:
            p, cap = ctypes.c_void_p(), ctypes.c_size_t()
            self._check(self._lib.pgb_stream_buffer(self._h, k, ctypes.byref(p), ctypes.byref(cap)))
            nbytes = chunks[k].length * C
            buf = (ctypes.c_uint8 * nbytes).from_address(p.value)
            mv = memoryview(buf).cast("B")
            off0 = data_offset + chunks[k].start_sample * C
            step = -(-nbytes // max(1, read_threads))

            def rd(a: int) -> None:
                b = min(nbytes, a + step)
                while a < b:
                    n = os.preadv(fd, [mv[a:b]], off0 + a)
                    if n <= 0:
                        raise OSError(f"short read at byte {off0 + a}")
                    a += n

            list(pool.map(rd, range(0, nbytes, step)))
            # start the upload now: it overlaps the previous chunk's compute
            self._check(self._lib.pgb_stream_upload(self._h, k))

        def piece(j: int, npieces: int, mv, off0: int, nbytes: int) -> None:
            """Piece j of chunk 0 (its rows as the library splits them), uploaded when read."""
            L = chunks[0].length

            def row(i: int) -> int:  # the library's piece boundaries (pgb_stream_upload_part)
                return L if i >= npieces else L * i // npieces // 64 * 64

            a, b = row(j) * C, row(j + 1) * C
            ok = 0
            try:
                while a < b:
                    n = os.preadv(fd, [mv[a:b]], off0 + a)
                    if n <= 0:
                        raise OSError(f"short read at byte {off0 + a}")
                    a += n
                ok = 1
            finally:
                self._check(self._lib.pgb_stream_upload_part(self._h, 0, j, npieces, ok))

        import time

        t_read = 0.0
        t0 = time.perf_counter()
        # chunk 0 is read and uploaded piece by piece and its tiles computed as the rows
        # arrive (RFI excision needs whole chunks)
        progressive = bool(chunks) and rc is None
        try:
            with ThreadPoolExecutor(1) as reader:
                pieces = []
                if progressive:
                    p, cap = ctypes.c_void_p(), ctypes.c_size_t()
                    self._check(self._lib.pgb_stream_buffer(self._h, 0, ctypes.byref(p), ctypes.byref(cap)))
                    nb0 = chunks[0].length * C
                    mv0 = memoryview((ctypes.c_uint8 * nb0).from_address(p.value)).cast("B")
                    npieces = max(2, read_threads)
                    off0 = data_offset + chunks[0].start_sample * C
                    # announce the pieces, so the push below waits for them
                    self._check(self._lib.pgb_stream_upload_part(self._h, 0, 0, npieces, -1))
                    pieces = [pool.submit(piece, j, npieces, mv0, off0, nb0) for j in range(npieces)]
                    fut = reader.submit(fill, 1) if len(chunks) > 1 else None
                else:
                    fut = reader.submit(fill, 0) if chunks else None
                for k in range(len(chunks)):
                    if not (progressive and k == 0):
                        tw = time.perf_counter()
                        fut.result()  # waiting here = the reader is behind the device
                        t_read += time.perf_counter() - tw
                        if k + 1 < len(chunks):
                            fut = reader.submit(fill, k + 1)
                    self._check(self._lib.pgb_stream_push(self._h, k, None))
                    if progressive and k == 0:
                        for f in pieces:
                            f.result()
        finally:
            pool.shutdown()
        nc, ncl = ctypes.c_size_t(), ctypes.c_size_t()
        self._check(self._lib.pgb_stream_finish(self._h, ctypes.byref(nc), ctypes.byref(ncl)))
        total = time.perf_counter() - t0
        cms = ctypes.c_double()
        self._check(self._lib.pgb_last_cluster_ms(self._h, ctypes.byref(cms)))
        self._stream_times = {"read_ms": 1e3 * t_read, "cluster_ms": cms.value,
                              "dm_loop_ms": 1e3 * (total - t_read) - cms.value}
        return self.fetch_file_results(nc.value, ncl.value)

    def last_stream_times(self) -> dict:
        """Host-clock stage times of the last search_stream (FileOutcome fields)."""
        return dict(self._stream_times)

    def copy_async(self, dst: int, src: int, nbytes: int) -> None:
        """cudaMemcpyAsync on this context's stream (host, device or peer pointers)."""
        self._check(self._lib.pgb_copy_async(self._h, ctypes.c_void_p(dst), ctypes.c_void_p(src), int(nbytes)))

    def synchronize(self) -> None:
        self._check(self._lib.pgb_synchronize(self._h))

    # ---- RFI excision --------------------------------------------------------------------
    def rfi_clean(self, chunk_data: np.ndarray, plan: DmTrialPlan, rfi: RfiConfig):
        """flag_narrowband + flag_broadband + apply_mask (src/rfi.cpp:32-139) on one chunk.

        Returns (cleaned float chunk, bad-channel mask, bad-sample mask)."""
        self.set_plan(plan)
        data = np.asarray(chunk_data)
        is_u8 = data.dtype == np.uint8
        data = np.ascontiguousarray(data, dtype=np.uint8 if is_u8 else np.float32)
        L, nch = data.shape
        out = np.zeros((L, nch), np.float32)
        rc = rfi._c()
        nbc, nbs = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._lib.pgb_rfi_clean(self._h, abi.ptr(data), int(is_u8), 0, L, ctypes.byref(rc), abi.ptr(out),
                                ctypes.byref(nbc), ctypes.byref(nbs)))
        bc = np.zeros(nch, np.uint8)
        bs = np.zeros(L, np.uint8)
        self._check(self._lib.pgb_fetch_rfi_flags(self._h, abi.ptr(bc), abi.ptr(bs)))
        return out, bc.astype(bool), bs.astype(bool)

    def fetch_file_results(self, nc: int, ncl: int):
        cands = np.zeros(nc, abi.CANDIDATE_DTYPE)
        self._check(self._lib.pgb_fetch_file_candidates(self._h, abi.ptr(cands), nc))
        clusters = self._fetch_clusters(ncl, nc)
        npairs = ctypes.c_size_t()
        self._check(self._lib.pgb_fetch_file_skipped(self._h, None, 0, ctypes.byref(npairs)))
        pairs = np.zeros((npairs.value, 2), np.uint64)
        self._check(self._lib.pgb_fetch_file_skipped(self._h, abi.ptr(pairs), npairs.value, ctypes.byref(npairs)))
        return cands, clusters, pairs

    # ---- instrumentation ------------------------------------------------------------------
    def launch_count(self) -> int:
        v = ctypes.c_uint64()
        self._check(self._lib.pgb_launch_count(self._h, ctypes.byref(v)))
        return v.value

    def last_dedisp_time(self) -> tuple[float, int, int]:
        ms, n, adds = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._lib.pgb_last_dedisp_time(self._h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(adds)))
        return ms.value, n.value, adds.value

    def stream_handle(self) -> int:
        p = ctypes.c_void_p()
        self._check(self._lib.pgb_stream(self._h, ctypes.byref(p)))
        return p.value or 0


_engines: dict[tuple[int, int], Engine] = {}
_lock = threading.Lock()


def default_engine(device: int = 0) -> Engine:
    """One engine per (thread, device): run_dm_loop is re-entrant across threads like the
    reference's (src/pipeline.cpp:182-194)."""
    key = (threading.get_ident(), device)
    with _lock:
        eng = _engines.get(key)
        if eng is None:
            eng = _engines[key] = Engine(device)
        return eng


_idle: dict[int, list[Engine]] = {}


def acquire_engine(device: int = 0) -> Engine:
    """An idle device context from the process-wide pool (created on first use).  The
    multi-file workers take one per file batch and hand it back, so contexts, streams and
    their grown device arenas outlive a batch instead of paying cudaMalloc per call."""
    with _lock:
        free = _idle.setdefault(device, [])
        if free:
            return free.pop()
    return Engine(device)


def release_engine(eng: Engine) -> None:
    with _lock:
        _idle.setdefault(eng.device, []).append(eng)


def run_dm_loop(chunk: Chunk, plan: DmTrialPlan, cfg: EngineConfig, pool=None, *,
                device: int = 0) -> DmLoopResult:
    """pulsegrid::run_dm_loop (engine.hpp:61-62) on the B200."""
    return default_engine(device).run_dm_loop(chunk, plan, cfg, pool)
