"""Deterministic synthetic 8-bit filterbanks for the benchmark and the full-size parity tests.

TEST / BENCHMARK INFRASTRUCTURE (not product code).  The bytes of a file depend only on
the config dict (shape, seed, pulses, RFI switch), never on the machine or the thread
count, so the dev container (where the reference library produces the golden
candidates, tests/golden/make_golden_configs.py) and the GPU box (where the device
path is checked against them) see identical payloads without shipping gigabytes.

* Noise: N(100, 16^2) quantised round-half-up to u8 (the value distribution of
  SURVEY.md section 8(d)), drawn through an inverse-CDF table from uniform u16 codes.
  Rows are generated in 4096-row blocks, block b from PCG64(SeedSequence([seed, b])),
  so any row range (one chunk) is reproducible without generating the whole file,
  and blocks generate in parallel threads.
* Pulses: dispersed top-hats along the plan's own delays for the chosen trial
  (amplitude snr*sigma/sqrt(nchans*width), the reference's amplitude_for_snr,
  src/synth.cpp:77-80), added per cell with round-half-up and clamping.
* RFI (config E): 5 % hot channels (+40) and 2-row DM-0 bursts (+30) every 4096 rows.
"""
from __future__ import annotations

import math
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from functools import lru_cache
from pathlib import Path

import numpy as np

BLOCK_ROWS = 4096

# BASELINE.json configs; SURVEY.md section 8(d) table.  C1 / E1 are one-chunk files
# of the C / E bands (the full-size golden cases; the full C file is 2^22 samples).
CONFIGS = {
    "A": dict(workload="config_A", nchans=1024, fch1=1500.0, foff=-0.25, tsamp=64e-6,
              nsamples=1 << 16, dm_lo=0.0, dm_hi=500.0, dm_step=2.0, boxcar_max=4096,
              detect_thresh=6.0, baseline_s=2.0, nsamps_chunk=1 << 18, npulses=3, seed=1000),
    "B": dict(workload="config_B_parkes_like", nchans=4096, fch1=1518.0, foff=-0.0703125,
              tsamp=64e-6, nsamples=1 << 20, dm_lo=0.0, dm_hi=2000.0, dm_step=2.0,
              boxcar_max=4096, detect_thresh=6.0, baseline_s=2.0, nsamps_chunk=1 << 18,
              npulses=10, seed=1001),
    "C": dict(workload="config_C_fast_like", nchans=4096, fch1=1500.0, foff=-0.1220703125,
              tsamp=49.152e-6, nsamples=1 << 22, dm_lo=0.0, dm_hi=5000.0, dm_step=1.25,
              boxcar_max=4096, detect_thresh=6.0, baseline_s=2.0, nsamps_chunk=1 << 20,
              npulses=8, seed=3000),
    "E": dict(workload="config_E_rfi_stress", nchans=8192, fch1=1500.0, foff=-0.0625,
              tsamp=64e-6, nsamples=1 << 20, dm_lo=0.0, dm_hi=2047.5, dm_step=0.5,
              boxcar_max=4096, detect_thresh=6.0, baseline_s=2.0, nsamps_chunk=1 << 19,
              npulses=50, seed=5000, rfi=True),
}
CONFIGS["C1"] = dict(CONFIGS["C"], workload="config_C_one_chunk", nsamples=1 << 20, seed=3001)
CONFIGS["E1"] = dict(CONFIGS["E"], workload="config_E_one_chunk", nsamples=1 << 19, seed=5001)


@lru_cache(maxsize=None)
def noise_table(mean: float = 100.0, sigma: float = 16.0) -> np.ndarray:
    """u16 code -> N(mean, sigma^2) quantised round-half-up to u8 (inverse CDF at bin centres)."""
    from statistics import NormalDist

    nd = NormalDist(mean, sigma)
    u = (np.arange(65536) + 0.5) / 65536.0
    x = np.array([nd.inv_cdf(float(v)) for v in u])
    return np.clip(np.floor(x + 0.5), 0, 255).astype(np.uint8)


def _noise_block(seed: int, b: int, nchans: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(b)])))
    codes = np.frombuffer(rng.bytes(2 * BLOCK_ROWS * nchans), dtype="<u2")
    return noise_table()[codes].reshape(BLOCK_ROWS, nchans)


def noise(nchans: int, seed: int, row0: int, rows: int, out: np.ndarray | None = None,
          threads: int | None = None) -> np.ndarray:
    """Rows [row0, row0+rows) of the seed's noise field as [rows][nchans] u8."""
    if out is None:
        out = np.empty((rows, nchans), np.uint8)
    b0, b1 = row0 // BLOCK_ROWS, (row0 + rows + BLOCK_ROWS - 1) // BLOCK_ROWS

    def fill(b):
        blk = _noise_block(seed, b, nchans)
        lo, hi = max(row0, b * BLOCK_ROWS), min(row0 + rows, (b + 1) * BLOCK_ROWS)
        out[lo - row0: hi - row0] = blk[lo - b * BLOCK_ROWS: hi - b * BLOCK_ROWS]

    with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, range(b0, b1)))
    return out


def pulse_specs(cfg: dict, delays: np.ndarray) -> list[tuple[int, int, int, float]]:
    """(trial, t0, width, snr) of the injected pulses, spread over DM, time and width."""
    rng = np.random.default_rng(cfg["seed"])
    ntrials = delays.shape[0]
    out = []
    n = cfg["npulses"]
    for k in range(n):
        trial = int((k + 0.5) / n * (ntrials - 1))
        width = 1 << int(rng.integers(0, 8))
        snr = float(rng.uniform(12.0, 20.0))
        span = cfg["nsamples"] - int(delays[trial].max()) - width - 1
        t0 = int((k + 0.5) / n * span)
        out.append((trial, t0, width, snr))
    return out


def inject_pulses(block: np.ndarray, row0: int, cfg: dict, delays: np.ndarray, sigma: float = 16.0):
    """Add the config's pulses to the rows [row0, row0+len(block)) held in `block`."""
    rows, nch = block.shape
    chans = np.arange(nch)
    for trial, t0, width, snr in pulse_specs(cfg, delays):
        amp = snr * sigma / math.sqrt(nch * width)
        d = delays[trial].astype(np.int64)
        for w in range(width):
            r = t0 + d + w - row0
            keep = (r >= 0) & (r < rows)
            rr, cc = r[keep], chans[keep]
            v = block[rr, cc].astype(np.float64) + amp
            block[rr, cc] = np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8)


def add_rfi(block: np.ndarray, row0: int, cfg: dict):
    """Config E's dense RFI: 5 % hot channels (+40) and 2-row DM-0 bursts (+30) every 4096 rows."""
    rows, nch = block.shape
    n = cfg["nsamples"]
    hot = np.sort(np.random.default_rng(cfg["seed"]).choice(nch, nch // 20, replace=False))
    block[:, hot] = np.minimum(block[:, hot].astype(np.int16) + 40, 255).astype(np.uint8)
    for t in range(2048, n - 2, 4096):
        for r in (t, t + 1):
            if row0 <= r < row0 + rows:
                block[r - row0] = np.minimum(block[r - row0].astype(np.int16) + 30, 255).astype(np.uint8)


def payload(cfg: dict, delays: np.ndarray, row0: int = 0, rows: int | None = None,
            out: np.ndarray | None = None) -> np.ndarray:
    """Rows [row0, row0+rows) (default: the whole file) of the config's 8-bit payload."""
    rows = cfg["nsamples"] - row0 if rows is None else rows
    blk = noise(cfg["nchans"], cfg["seed"], row0, rows, out=out)
    inject_pulses(blk, row0, cfg, delays)
    if cfg.get("rfi"):
        add_rfi(blk, row0, cfg)
    return blk


def header_bytes(cfg: dict, source_name: str = "pgsynth", tstart: float = 60000.0) -> bytes:
    """SIGPROC header in the reference writer's keyword order (src/filterbank.cpp:186-211)."""

    def s(x: str) -> bytes:
        b = x.encode()
        return struct.pack("<i", len(b)) + b

    h = s("HEADER_START") + s("source_name") + s(source_name)
    h += s("telescope_id") + struct.pack("<i", 0) + s("machine_id") + struct.pack("<i", 0)
    h += s("data_type") + struct.pack("<i", 1)
    h += s("fch1") + struct.pack("<d", cfg["fch1"]) + s("foff") + struct.pack("<d", cfg["foff"])
    h += s("nchans") + struct.pack("<i", cfg["nchans"]) + s("nbits") + struct.pack("<i", 8)
    h += s("tstart") + struct.pack("<d", tstart) + s("tsamp") + struct.pack("<d", cfg["tsamp"])
    h += s("nifs") + struct.pack("<i", 1) + s("HEADER_END")
    return h


def write_filterbank(path: str | Path, cfg: dict, delays: np.ndarray, rows_per_write: int = 1 << 16):
    """Write the config's file (header + raw u8 payload) without holding it all in memory."""
    with open(path, "wb") as f:
        f.write(header_bytes(cfg))
        for r0 in range(0, cfg["nsamples"], rows_per_write):
            r = min(rows_per_write, cfg["nsamples"] - r0)
            f.write(payload(cfg, delays, r0, r).tobytes())
