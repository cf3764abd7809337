"""Golden outputs of the reference pipeline at the BASELINE.json config shapes.

TEST INFRASTRUCTURE.  Run in the dev container (needs oracle/_ref, i.e. the reference
library compiled from /root/reference):

    python tests/golden/make_golden_configs.py [A B C1 E1] [--threads N]

For each config the deterministic payload of tools/synth.py is written as an 8-bit
SIGPROC file and searched by the UNMODIFIED reference pipeline in parity mode
(oracle/ref_harness.cpp `pgref_search_file`: create_task, FilterbankReader::read_chunk,
flag_narrowband/flag_broadband/apply_mask when RFI is on, run_dm_loop with
max_in_flight == n_workers, the file-level sort and link_grid,
src/pipeline.cpp:32-119).  The results land in tests/golden/config_<name>.npz:

* the sha256 of the payload bytes (pins the generator: the GPU box regenerates the
  file and checks the digest before comparing anything);
* the full sorted candidate list (every field, snr included) when it is small enough
  to commit, otherwise per-field sha256 digests plus the count;
* the clusters, their member ids, the skipped (chunk, trial) pairs and the .cand text.

Configs: A = the full config-A file; B = the full config-B file (5 chunks, ~8 min on 8
cores); C1 = one 2^20-sample file of the config-C band with all 4001 trials; E1 = one
2^19-sample file of the config-E band, 4096 trials, dense RFI with RFI excision on.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Reference  # noqa: E402
from tools import synth  # noqa: E402

MAX_INLINE = 150_000  # candidates stored in full below this count


def file_digest(cfg: dict, delays: np.ndarray, rows: int = 1 << 16) -> str:
    h = hashlib.sha256()
    for r0 in range(0, cfg["nsamples"], rows):
        h.update(synth.payload(cfg, delays, r0, min(rows, cfg["nsamples"] - r0)).tobytes())
    return h.hexdigest()


def field_digests(c: np.ndarray) -> dict:
    return {k: hashlib.sha256(np.ascontiguousarray(c[k]).tobytes()).hexdigest() for k in c.dtype.names}


def run(name: str, threads: int, workdir: Path) -> dict:
    cfg = dict(synth.CONFIGS[name])
    ref = Reference()
    dms, delays = ref.generate_dm_trials(cfg["dm_lo"], cfg["dm_hi"], cfg["fch1"], cfg["foff"], cfg["tsamp"],
                                         cfg["nchans"], step=cfg["dm_step"])
    path = workdir / f"{name}.fil"
    t0 = time.time()
    synth.write_filterbank(path, cfg, delays)
    digest = file_digest(cfg, delays)
    print(f"[{name}] wrote {path} ({path.stat().st_size / 2**30:.2f} GiB) in {time.time() - t0:.0f}s",
          flush=True)
    rfi = bool(cfg.get("rfi"))
    t0 = time.time()
    res = ref.search_file(path, dm_lo=cfg["dm_lo"], dm_hi=cfg["dm_hi"], dm_step=cfg["dm_step"],
                          n_workers=threads, detect_thresh=cfg["detect_thresh"],
                          boxcar_max=cfg["boxcar_max"], baseline_len_s=cfg["baseline_s"],
                          nsamps_chunk=cfg["nsamps_chunk"], rfi_narrowband=rfi, rfi_broadband=rfi,
                          parity=True)
    wall = time.time() - t0
    cands = res["candidates"]
    meta = dict(config=name, cfg=cfg, payload_sha256=digest, ncandidates=int(len(cands)),
                nclusters=int(len(res["clusters"])), nskipped=int(len(res["skipped"])),
                threads=threads, wall_s=wall, stage_ms=res["stage_ms"],
                candidate_digests=field_digests(cands), ntrials=int(len(dms)))
    out = dict(meta=json.dumps(meta), clusters=res["clusters"], members=res["members"],
               skipped=res["skipped"], cand_text=np.frombuffer(res["cand_text"].encode(), np.uint8))
    if len(cands) <= MAX_INLINE:
        out["candidates"] = cands
    np.savez_compressed(HERE / f"config_{name}.npz", **out)
    print(f"[{name}] {len(cands)} candidates, {len(res['clusters'])} clusters, "
          f"{len(res['skipped'])} skipped; reference search {wall:.0f}s on {threads} threads", flush=True)
    path.unlink()
    return meta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["A", "B", "C1", "E1"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--workdir", default="/tmp/pg_golden")
    args = ap.parse_args()
    wd = Path(args.workdir)
    wd.mkdir(parents=True, exist_ok=True)
    for name in args.configs:
        run(name, args.threads, wd)


if __name__ == "__main__":
    main()
