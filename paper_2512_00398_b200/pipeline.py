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


def run_multi_file(payloads: list[np.ndarray], tasks: list[SearchTask], *, n_exec: int = 4,
                   device: int = 0) -> list[SearchResult | Exception]:
    """Multi-file execution (src/pipeline.cpp:136-210, next row f3) on one GPU.

    The reference overlaps task creation and execution with two bounded queues of
    worker threads; here `n_exec` host threads each own a device context (its own
    CUDA stream and arena, `default_engine` is per thread), so several files'
    uploads, kernels and syncs interleave on the GPU.  Results are in submission
    order; a failing file yields its exception instead of a result (per-file
    isolation, src/pipeline.cpp:173-192)."""
    from concurrent.futures import ThreadPoolExecutor

    if n_exec < 1:
        from .errors import ConfigError

        raise ConfigError("need at least one worker per stage")

    def one(k):
        try:
            return search_file(payloads[k], tasks[k], device=device)
        except Exception as exc:  # isolate-and-continue
            return exc

    with ThreadPoolExecutor(n_exec) as ex:
        return list(ex.map(one, range(len(tasks))))


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


def search_fil(path: str | Path, params: SearchParams, *, device: int = 0, read_threads: int = 4,
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
