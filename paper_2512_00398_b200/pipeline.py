"""File-level search around the hot path: execute_task's chunk loop on raw 8-bit data.

Mirrors the caller side of the path (/root/reference/proj/src/pipeline.cpp:22-119):
`create_task` resolves the DM plan, baseline window and overlapping chunk plan
exactly like the reference; `search_file` then runs every chunk on the device
(raw u8 payload uploaded segment by segment on a copy stream),
sorts all candidates and clusters them with link_grid without leaving the GPU;
`write_candidates` produces the reference's .cand text (src/cluster_io.cpp:11-34).

RFI excision (src/rfi.cpp, next row f1) runs on the device before each chunk's
DM loop when enabled (`SearchParams.rfi`, reference defaults: both flaggers on,
local-mean replacement).
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .dedisp import DmTrialPlan, FilterbankHeader, LinearSpacing, AdaptiveSpacing, generate_dm_trials
from .engine import ChunkSpec, EngineConfig, RfiConfig, default_engine
from .cluster import Clusters


def plan_chunks(nsamples: int, chunk_len: int, overlap: int) -> list[ChunkSpec]:
    """src/filterbank.cpp:239-272."""
    from .errors import InvalidPlanError

    if nsamples == 0:
        raise InvalidPlanError("empty file")
    if chunk_len == 0:
        raise InvalidPlanError("chunk_len must be positive")
    if overlap >= chunk_len:
        raise InvalidPlanError(f"overlap {overlap} must be smaller than chunk_len {chunk_len}")
    if chunk_len >= nsamples:
        return [ChunkSpec(0, 0, nsamples, 0, 0, nsamples)]
    stride = chunk_len - overlap
    plan: list[ChunkSpec] = []
    start = 0
    while True:
        if start + chunk_len >= nsamples:
            plan.append(ChunkSpec(len(plan), start, nsamples - start, 0, start, nsamples))
            return plan
        plan.append(ChunkSpec(len(plan), start, chunk_len, overlap, start, start + stride))
        start += stride


def baseline_window_samples(baseline_len_s: float, tsamp: float) -> int:
    """src/pipeline.cpp:22-28 (llround, forced odd)."""
    if baseline_len_s <= 0.0:
        return 0
    x = baseline_len_s / tsamp
    w = int(math.floor(x + 0.5)) if x >= 0 else int(math.ceil(x - 0.5))
    w = max(w, 1)
    return w + 1 if w % 2 == 0 else w


@dataclass
class SearchParams:
    """pulsegrid::SearchParams (pipeline.hpp:17-38), the fields the path uses."""

    dm_lo: float = 0.0
    dm_hi: float = 1000.0
    spacing: LinearSpacing | AdaptiveSpacing = field(default_factory=lambda: AdaptiveSpacing(1.25))
    engine: EngineConfig = field(default_factory=EngineConfig)
    baseline_len_s: float = 2.0
    nsamps_chunk: int = 1 << 18
    rfi: RfiConfig = field(default_factory=RfiConfig)  # reference default: both flaggers on


@dataclass
class SearchTask:
    """pulsegrid::PipelineTask (pipeline.hpp:41-50) minus I/O state."""

    header: FilterbankHeader
    plan: DmTrialPlan
    engine: EngineConfig
    chunks: list[ChunkSpec]
    rfi: RfiConfig = field(default_factory=lambda: RfiConfig(False, False))


def create_task(header: FilterbankHeader, params: SearchParams) -> SearchTask:
    """src/pipeline.cpp:32-59 (without opening the file)."""
    from .errors import PulsegridError

    if header.nsamples == 0:
        raise PulsegridError("file has no samples")
    plan = generate_dm_trials(params.dm_lo, params.dm_hi, header, params.spacing)
    eng = EngineConfig(**{k: getattr(params.engine, k) for k in params.engine.__dataclass_fields__})
    eng.tsamp = header.tsamp
    eng.baseline_window = baseline_window_samples(params.baseline_len_s, header.tsamp)
    overlap = plan.max_delay + params.engine.boxcar_max
    chunk_len = params.nsamps_chunk
    if chunk_len <= overlap or header.nsamples <= overlap:
        chunk_len = header.nsamples
    chunks = plan_chunks(header.nsamples, chunk_len, 0 if chunk_len >= header.nsamples else overlap)
    return SearchTask(header, plan, eng, chunks, params.rfi)


@dataclass
class SearchResult:
    candidates: np.ndarray          # all chunks, sorted (peak, trial, width)
    clusters: Clusters              # link_grid of the candidates
    skipped: np.ndarray             # [k, 2] (chunk index, trial)


def search_file(payload: np.ndarray, task: SearchTask, *, device: int = 0,
                trial_range: tuple[int, int] | None = None) -> SearchResult:
    """execute_task's loop (src/pipeline.cpp:72-106) on a [nsamples][nchans] u8 payload."""
    eng = default_engine(device)
    cands, clusters, skipped = eng.search_file(payload, task.header.nsamples, task.chunks,
                                               task.plan, task.engine, trial_range=trial_range,
                                               rfi=task.rfi)
    return SearchResult(cands, clusters, skipped)


def search_payloads(payloads: list[np.ndarray], tasks: list[SearchTask], *, n_exec: int = 4,
                    devices: tuple[int, ...] = (0,)) -> list[SearchResult | Exception]:
    """In-memory multi-file search (config D without disk I/O): `n_exec` host threads, each
    owning one device context (worker k on devices[k % len(devices)]), take files in
    submission order; a failing file yields its exception instead of a result."""
    import queue
    import threading

    from .engine import acquire_engine, release_engine
    from .errors import ConfigError

    if n_exec < 1:
        raise ConfigError("need at least one worker per stage")
    out: list[SearchResult | Exception | None] = [None] * len(tasks)
    q: queue.Queue = queue.Queue()
    for k in range(len(tasks)):
        q.put(k)

    def worker(w: int) -> None:
        eng = acquire_engine(devices[w % len(devices)])
        try:
            while True:
                try:
                    k = q.get_nowait()
                except queue.Empty:
                    return
                try:
                    t = tasks[k]
                    c, cl, sk = eng.search_file(payloads[k], t.header.nsamples, t.chunks, t.plan, t.engine,
                                                rfi=t.rfi)
                    out[k] = SearchResult(c, cl, sk)
                except Exception as exc:  # isolate-and-continue (src/pipeline.cpp:183-190)
                    out[k] = exc
        finally:
            release_engine(eng)

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(n_exec)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return out  # type: ignore[return-value]


# ---- multi-file pipeline (src/pipeline.cpp:121-219, include/pulsegrid/pipeline.hpp:52-96) ----

@dataclass
class FileOutcome:
    """pulsegrid::FileOutcome (pipeline.hpp:52-65): per-file status and stage times (ms)."""

    path: str = ""
    output_path: str = ""
    ok: bool = False
    error: str = ""
    candidates: int = 0                    # clusters written
    wall_ms: float = 0.0
    skipped_trials: list[tuple[int, int]] = field(default_factory=list)  # (chunk, trial)
    read_ms: float = 0.0                   # waiting for chunk bytes (reader behind compute)
    rfi_ms: float = 0.0                    # device RFI is inside dm_loop_ms (one stream)
    dm_loop_ms: float = 0.0
    cluster_ms: float = 0.0
    write_ms: float = 0.0
    device: int = 0


@dataclass
class RunSummary:
    """pulsegrid::RunSummary (pipeline.hpp:67-71)."""

    files: list[FileOutcome]
    total_wall_ms: float = 0.0
    n_failed: int = 0


def assign_output_paths(paths: list[str], output_dir: str) -> list[str]:
    """src/pipeline.cpp:121-133: <output_dir>/<stem>.cand, repeated stems numbered."""
    seen: dict[str, int] = {}
    out = []
    for p in paths:
        stem = Path(p).stem or "output"
        seen[stem] = seen.get(stem, 0) + 1
        n = seen[stem]
        out.append(str(Path(output_dir) / (f"{stem}.cand" if n == 1 else f"{stem}.{n}.cand")))
    return out


@dataclass
class PipelineTask:
    """pulsegrid::PipelineTask (pipeline.hpp:41-50)."""

    index: int
    path: str
    output_path: str
    task: SearchTask
    data_offset: int


def create_file_task(path: str, params: SearchParams, output_path: str, index: int = 0) -> PipelineTask:
    """create_task on a file (src/pipeline.cpp:32-59): header, DM plan, chunk plan."""
    from .errors import PulsegridError

    hdr, off = read_filterbank_header(path)
    if hdr.nsamples == 0:
        raise PulsegridError(f"'{path}' has no samples")
    return PipelineTask(index, str(path), output_path, create_task(hdr, params), off)


def execute_task(pt: PipelineTask, eng, read_threads: int = 8) -> FileOutcome:
    """execute_task (src/pipeline.cpp:61-119) on the device: streamed chunks (bounded memory),
    the chunk chain, file sort + link_grid, one .cand file; stage times in the outcome."""
    import os
    import time

    t0 = time.perf_counter()
    out = FileOutcome(path=pt.path, output_path=pt.output_path, device=eng.device)
    fd = os.open(pt.path, os.O_RDONLY)
    try:
        t = pt.task
        c, cl, sk = eng.search_stream(fd, pt.data_offset, t.header.nsamples, t.chunks, t.plan, t.engine,
                                      rfi=t.rfi, read_threads=read_threads)
    finally:
        os.close(fd)
    st = eng.last_stream_times()
    out.read_ms, out.dm_loop_ms, out.cluster_ms = st["read_ms"], st["dm_loop_ms"], st["cluster_ms"]
    tw = time.perf_counter()
    text = write_candidates(cl)
    with open(pt.output_path, "w") as f:
        f.write(text)
    out.write_ms = 1e3 * (time.perf_counter() - tw)
    out.candidates = len(cl)
    out.skipped_trials = [(int(a), int(b)) for a, b in np.asarray(sk).reshape(-1, 2)]
    out.ok = True
    out.wall_ms = 1e3 * (time.perf_counter() - t0)
    return out


def run_multi_file(paths: list[str], params: SearchParams, output_dir: str, n_create: int = 1,
                   n_exec: int = 2, creation_capacity: int = 0, execution_capacity: int = 0, *,
                   devices: tuple[int, ...] = (0,), read_threads: int = 8) -> RunSummary:
    """Two-stage multi-file pipeline (src/pipeline.cpp:136-210): n_create workers parse
    headers and build plans, n_exec workers execute them through bounded queues (capacity
    2x the stage's workers by default), per-file failures isolated into the summary.  Each
    execution worker owns one device context; worker k runs on devices[k % len(devices)],
    so a batch spreads over the node's GPUs.  The memory budget is split across the
    execution workers like the reference's (:163-166)."""
    import queue
    import threading
    import time

    from .engine import acquire_engine, release_engine
    from .errors import ConfigError

    if n_create < 1 or n_exec < 1:
        raise ConfigError("need at least one worker per stage")
    t0 = time.perf_counter()
    Path(output_dir).mkdir(parents=True, exist_ok=True)
    outs = assign_output_paths([str(p) for p in paths], output_dir)
    summary = RunSummary([FileOutcome(path=str(p), output_path=o) for p, o in zip(paths, outs)])
    wp = SearchParams(**{k: getattr(params, k) for k in params.__dataclass_fields__})
    wp.engine = EngineConfig(**{k: getattr(params.engine, k) for k in params.engine.__dataclass_fields__})
    wp.engine.memory_budget = max(1, params.engine.memory_budget // n_exec)
    cq: queue.Queue = queue.Queue(creation_capacity or 2 * n_create)
    eq: queue.Queue = queue.Queue(execution_capacity or 2 * n_exec)
    STOP = object()

    def creator():
        while (item := cq.get()) is not STOP:
            try:
                eq.put(create_file_task(str(paths[item]), wp, outs[item], item))
            except Exception as exc:
                summary.files[item].ok = False
                summary.files[item].error = str(exc)

    def executor(w: int):
        eng = acquire_engine(devices[w % len(devices)])
        try:
            while (pt := eq.get()) is not STOP:
                try:
                    summary.files[pt.index] = execute_task(pt, eng, read_threads)
                except Exception as exc:
                    summary.files[pt.index].ok = False
                    summary.files[pt.index].error = str(exc)
        finally:
            release_engine(eng)

    creators = [threading.Thread(target=creator) for _ in range(n_create)]
    executors = [threading.Thread(target=executor, args=(w,)) for w in range(n_exec)]
    for t in creators + executors:
        t.start()
    for i in range(len(paths)):
        cq.put(i)
    for _ in creators:
        cq.put(STOP)
    for t in creators:
        t.join()
    for _ in executors:  # creators done: drain and stop the executors
        eq.put(STOP)
    for t in executors:
        t.join()
    summary.n_failed = sum(not f.ok for f in summary.files)
    summary.total_wall_ms = 1e3 * (time.perf_counter() - t0)
    return summary


def write_summary(summary: RunSummary) -> str:
    """src/pipeline.cpp:212-219: path, status, candidate count, wall ms (+ error)."""
    lines = []
    for f in summary.files:
        line = f"{f.path}\t{'ok' if f.ok else 'error'}\t{f.candidates}\t{int(round(f.wall_ms))}"
        if not f.ok:
            line += f"\t{f.error}"
        lines.append(line + "\n")
    return "".join(lines)


def write_candidates(clusters: Clusters) -> str:
    """src/cluster_io.cpp:11-34: one line per cluster, sorted by (peak_sample, dm_trial)."""
    recs = clusters.records
    order = sorted(range(len(recs)), key=lambda k: (int(recs["representative"]["peak_sample"][k]),
                                                    int(recs["representative"]["dm_trial"][k]), k))
    lines = []
    for k in order:
        r = recs["representative"][k]
        lines.append("%.2f\t%d\t%.9f\t%d\t%d\t%.3f\t%d\t%d\t%d\n" % (
            float(r["snr"]), int(r["peak_sample"]), float(r["time_s"]), int(r["width_index"]),
            int(r["dm_trial"]), float(r["dm"]), int(recs["members"][k]),
            int(recs["begin_sample"][k]), int(recs["end_sample"][k])))
    return "".join(lines)


# ---- SIGPROC input (raw u8 ingest; src/filterbank.cpp:102-175) -------------------------

_INT_KEYS = {"telescope_id", "machine_id", "data_type", "nchans", "nbits", "nifs", "nsamples",
             "barycentric", "pulsarcentric", "nbeams", "ibeam"}
_DBL_KEYS = {"fch1", "foff", "tsamp", "tstart", "az_start", "za_start", "src_raj", "src_dej",
             "refdm", "period"}
_STR_KEYS = {"source_name", "rawdatafile"}


def read_filterbank_header(path: str | Path) -> tuple[FilterbankHeader, int]:
    """SIGPROC header (src/filterbank.cpp:102-175) and the payload's byte offset; nsamples
    is derived from the file size like the reference (payload / bytes per sample)."""
    from .errors import PulsegridError

    path = Path(path)
    with open(path, "rb") as f:
        raw = f.read(1 << 16)
    size = path.stat().st_size
    pos = 0

    def rstr():
        nonlocal pos
        (n,) = struct.unpack_from("<i", raw, pos)
        if n < 0 or n > 256:
            raise PulsegridError(f"implausible string length {n}")
        s = raw[pos + 4: pos + 4 + n].decode()
        pos += 4 + n
        return s

    if rstr() != "HEADER_START":
        raise PulsegridError("missing HEADER_START sentinel")
    vals: dict[str, object] = {}
    while True:
        key = rstr()
        if key == "HEADER_END":
            break
        if key in _INT_KEYS:
            (vals[key],) = struct.unpack_from("<i", raw, pos)
            pos += 4
        elif key in _DBL_KEYS:
            (vals[key],) = struct.unpack_from("<d", raw, pos)
            pos += 8
        elif key in _STR_KEYS:
            vals[key] = rstr()
        elif key == "signed":
            pos += 1
        else:
            raise PulsegridError(f"unknown header keyword '{key}'")
    nchans, nbits = int(vals.get("nchans", 0)), int(vals.get("nbits", 0))
    if nbits != 8:
        raise PulsegridError(f"raw ingest needs nbits=8 (file has {nbits})")
    payload = size - pos
    if nchans <= 0 or payload % nchans:
        raise PulsegridError("payload is not a whole number of samples")
    hdr = FilterbankHeader(fch1=float(vals["fch1"]), foff=float(vals["foff"]), nchans=nchans,
                           tsamp=float(vals["tsamp"]), nbits=nbits, nsamples=payload // nchans,
                           source_name=str(vals.get("source_name", "")),
                           tstart=float(vals.get("tstart", 0.0)))
    return hdr, pos


def read_filterbank(path: str | Path) -> tuple[FilterbankHeader, np.ndarray]:
    """Header + the raw 8-bit payload as [nsamples][nchans] (no float widening; whole file
    in memory -- `search_fil` streams instead)."""
    hdr, off = read_filterbank_header(path)
    payload = np.fromfile(path, dtype=np.uint8, offset=off)
    return hdr, payload.reshape(-1, hdr.nchans)


def search_fil(path: str | Path, params: SearchParams, *, device: int = 0, read_threads: int = 8,
               trial_range: tuple[int, int] | None = None) -> SearchResult:
    """create_task + execute_task on an 8-bit SIGPROC file with bounded memory
    (src/pipeline.cpp:32-119): chunks are read straight into pinned buffers by parallel
    preads while the previous chunk computes; host and device hold two chunks."""
    import os

    hdr, off = read_filterbank_header(path)
    task = create_task(hdr, params)
    eng = default_engine(device)
    fd = os.open(str(path), os.O_RDONLY)
    try:
        cands, clusters, skipped = eng.search_stream(fd, off, hdr.nsamples, task.chunks, task.plan,
                                                     task.engine, trial_range=trial_range, rfi=task.rfi,
                                                     read_threads=read_threads)
    finally:
        os.close(fd)
    return SearchResult(cands, clusters, skipped)
