"""Throughput of the other BASELINE.json configs on one B200 (not the bench.py contract
line, which is config B): A, C (single-GPU, all 4001 trials), D (32 x A, concurrent
contexts) and E (8192 ch, 4096 trials, dense RFI, RFI excision on).

    python tools/bench_configs.py [A C D E] [--steps K]

Prints one JSON line per config: DM-trial*samples/s, x real time, dedispersion
T-adds/s and the fraction of the time spent in dedispersion.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from tools import synth  # noqa: E402
from paper_2512_00398_b200.engine import default_engine  # noqa: E402

CONFIGS = {k: v for k, v in synth.CONFIGS.items() if k in ("A", "C", "E", "E1")}


def run_file(cfg, steps, label=None):
    task = bench.build_task(cfg)
    payload = bench.make_payload(cfg, task.plan)
    torch.cuda.synchronize()
    eng = default_engine(0)
    eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)  # warm-up
    dd = 0.0
    adds = 0
    torch.cuda.synchronize()
    clk = bench.ClockSampler(0).__enter__()
    t0 = time.perf_counter()
    for _ in range(steps):
        cands, clusters, _ = eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine,
                                             rfi=task.rfi)
        ms, _, a = eng.last_dedisp_time()
        dd += ms
        adds += a
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / steps
    clk.__exit__(None, None, None)
    units = task.plan.ntrials * cfg["nsamples"]
    return {"config": label or cfg["workload"], "ntrials": task.plan.ntrials, "nchans": cfg["nchans"],
            "nsamples": cfg["nsamples"], "chunks": len(task.chunks), "rfi": bool(cfg.get("rfi")),
            "value": units / el, "unit": "DM-trial*samples/s", "x_realtime": cfg["nsamples"] * cfg["tsamp"] / el,
            "s_per_file": el, "dedisp_tadd_s": adds / (dd / 1e3) / 1e12 if dd else None,
            "dedisp_share": (dd / steps / 1e3) / el, "candidates": int(len(cands)),
            "clusters": int(len(clusters)), "clocks": clk.summary(),
            "timing": "host wall clock around synchronous file searches (payload resident)"}


def run_multi(steps, nfiles=32, n_exec=4):
    """Config D: 32 config-A files (seeds 2000+i) held in host memory, n_exec device contexts
    (one stream each) taking files concurrently (pipeline.search_payloads)."""
    from paper_2512_00398_b200.pipeline import search_payloads

    cfg = dict(CONFIGS["A"])
    task = bench.build_task(cfg)
    # host payloads in pinned memory (a reader would fill pinned buffers, as search_fil does)
    payloads = [torch.from_numpy(synth.payload(dict(cfg, seed=2000 + i), task.plan.delays)).pin_memory().numpy()
                for i in range(nfiles)]
    search_payloads(payloads, [task] * nfiles, n_exec=n_exec)  # warm-up
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        for _ in range(steps):
            res = search_payloads(payloads, [task] * nfiles, n_exec=n_exec)
        el = (time.perf_counter() - t0) / steps
    assert not any(isinstance(r, Exception) for r in res)
    units = nfiles * task.plan.ntrials * cfg["nsamples"]
    return {"config": "config_D_32xA", "files": nfiles, "n_exec": n_exec, "value": units / el,
            "unit": "DM-trial*samples/s", "x_realtime": nfiles * cfg["nsamples"] * cfg["tsamp"] / el,
            "s_per_batch": el, "clocks": clk.summary(),
            "timing": "host wall clock around the concurrent batch (host payloads, H2D included)"}


def run_multi_disk(steps, nfiles=32, n_exec=4, workdir="/tmp/pg_configD"):
    """Config D from disk: the 32 files written as 8-bit SIGPROC files, run_multi_file
    (2 creation + n_exec execution workers, streamed chunks, .cand files written)."""
    from paper_2512_00398_b200.pipeline import run_multi_file
    from tests.test_gpu_stream import _params

    cfg = dict(CONFIGS["A"])
    task = bench.build_task(cfg)
    Path(workdir).mkdir(parents=True, exist_ok=True)
    paths = []
    for i in range(nfiles):
        p = Path(workdir) / f"A{i:02d}.fil"
        synth.write_filterbank(p, dict(cfg, seed=2000 + i), task.plan.delays)
        paths.append(str(p))
    params = _params(cfg)
    run_multi_file(paths, params, workdir + "/out", n_create=2, n_exec=n_exec)  # warm-up (page cache)
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        for _ in range(steps):
            s = run_multi_file(paths, params, workdir + "/out", n_create=2, n_exec=n_exec)
        el = (time.perf_counter() - t0) / steps
    assert s.n_failed == 0
    units = nfiles * task.plan.ntrials * cfg["nsamples"]
    return {"config": "config_D_32xA_from_disk", "files": nfiles, "n_exec": n_exec, "value": units / el,
            "unit": "DM-trial*samples/s", "x_realtime": nfiles * cfg["nsamples"] * cfg["tsamp"] / el,
            "s_per_batch": el, "clocks": clk.summary(),
            "stage_ms_mean": {k: float(np.mean([getattr(f, k) for f in s.files]))
                              for k in ("read_ms", "dm_loop_ms", "cluster_ms", "write_ms", "wall_ms")},
            "timing": "host wall clock around run_multi_file (files in page cache)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["A", "D", "C", "E"])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--n-exec", type=int, default=4, help="config D: concurrent device contexts")
    args = ap.parse_args()
    for name in args.configs:
        if name == "D":
            out = run_multi(args.steps, n_exec=args.n_exec)
        elif name == "Ddisk":
            out = run_multi_disk(args.steps, n_exec=args.n_exec)
        elif name == "E1norfi":  # config E's geometry on the integer path (what RFI costs)
            out = run_file(dict(synth.CONFIGS["E1"], rfi=False), args.steps, label="config_E_one_chunk_no_rfi")
        else:
            out = run_file(dict(CONFIGS[name]), args.steps)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
