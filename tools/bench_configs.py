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
from paper_2512_00398_b200.engine import default_engine  # noqa: E402

CONFIGS = {
    "A": dict(workload="config_A", nchans=1024, fch1=1500.0, foff=-0.25, tsamp=64e-6, nsamples=1 << 16,
              dm_lo=0.0, dm_hi=500.0, dm_step=2.0, boxcar_max=4096, detect_thresh=6.0, baseline_s=2.0,
              nsamps_chunk=1 << 18, npulses=3, seed=1000),
    "C": dict(workload="config_C_fast_like", nchans=4096, fch1=1500.0, foff=-0.1220703125, tsamp=49.152e-6,
              nsamples=1 << 22, dm_lo=0.0, dm_hi=5000.0, dm_step=1.25, boxcar_max=4096, detect_thresh=6.0,
              baseline_s=2.0, nsamps_chunk=1 << 20, npulses=8, seed=3000),
    "E": dict(workload="config_E_rfi_stress", nchans=8192, fch1=1500.0, foff=-0.0625, tsamp=64e-6,
              nsamples=1 << 20, dm_lo=0.0, dm_hi=2047.5, dm_step=0.5, boxcar_max=4096, detect_thresh=6.0,
              baseline_s=2.0, nsamps_chunk=1 << 19, npulses=50, seed=5000, rfi=True),
}


def add_rfi(payload: torch.Tensor, cfg, rng):
    """Dense RFI for config E: 5% hot channels and DM-0 bursts every ~4096 samples."""
    n, nch = payload.shape
    hot = torch.from_numpy(rng.choice(nch, nch // 20, replace=False)).to(payload.device)
    payload[:, hot] = torch.clamp(payload[:, hot].to(torch.int16) + 40, 0, 255).to(torch.uint8)
    for t in range(2048, n - 2, 4096):
        payload[t: t + 2] = torch.clamp(payload[t: t + 2].to(torch.int16) + 30, 0, 255).to(torch.uint8)


def run_file(cfg, steps, label=None):
    task = bench.build_task(cfg)
    payload = bench.make_payload(cfg, task.plan)
    if cfg.get("rfi"):
        add_rfi(payload, cfg, np.random.default_rng(cfg["seed"]))
    torch.cuda.synchronize()
    eng = default_engine(0)
    eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)  # warm-up
    dd = 0.0
    adds = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        cands, clusters, _ = eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine,
                                             rfi=task.rfi)
        ms, _, a = eng.last_dedisp_time()
        dd += ms
        adds += a
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / steps
    units = task.plan.ntrials * cfg["nsamples"]
    return {"config": label or cfg["workload"], "ntrials": task.plan.ntrials, "nchans": cfg["nchans"],
            "nsamples": cfg["nsamples"], "chunks": len(task.chunks), "rfi": bool(cfg.get("rfi")),
            "value": units / el, "unit": "DM-trial*samples/s", "x_realtime": cfg["nsamples"] * cfg["tsamp"] / el,
            "s_per_file": el, "dedisp_tadd_s": adds / (dd / 1e3) / 1e12 if dd else None,
            "dedisp_share": (dd / steps / 1e3) / el, "candidates": int(len(cands)),
            "clusters": int(len(clusters)), "timing": "host wall clock around synchronous file searches"}


def run_multi(steps, nfiles=32, n_exec=4):
    """Config D: 32 config-A files, n_exec device contexts (one stream each) working concurrently."""
    cfg = dict(CONFIGS["A"])
    task = bench.build_task(cfg)
    payloads = []
    for i in range(nfiles):
        c = dict(cfg, seed=2000 + i)
        payloads.append(bench.make_payload(c, task.plan))
    torch.cuda.synchronize()

    def one(i):
        eng = default_engine(0)
        cands, clusters, _ = eng.search_file(payloads[i], cfg["nsamples"], task.chunks, task.plan, task.engine)
        return len(clusters)

    with ThreadPoolExecutor(n_exec) as ex:
        list(ex.map(one, range(nfiles)))  # warm-up (creates the per-thread contexts)
        t0 = time.perf_counter()
        for _ in range(steps):
            list(ex.map(one, range(nfiles)))
        el = (time.perf_counter() - t0) / steps
    units = nfiles * task.plan.ntrials * cfg["nsamples"]
    return {"config": "config_D_32xA", "files": nfiles, "n_exec": n_exec, "value": units / el,
            "unit": "DM-trial*samples/s", "x_realtime": nfiles * cfg["nsamples"] * cfg["tsamp"] / el,
            "s_per_batch": el, "timing": "host wall clock around the concurrent batch"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["A", "D", "C", "E"])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--n-exec", type=int, default=4, help="config D: concurrent device contexts")
    args = ap.parse_args()
    for name in args.configs:
        if name == "D":
            out = run_multi(args.steps, n_exec=args.n_exec)
        else:
            out = run_file(dict(CONFIGS[name]), args.steps)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
