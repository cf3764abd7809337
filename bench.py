#!/usr/bin/env python
"""Headline benchmark: single-pulse search throughput on BASELINE.json configs[1].

Workload (config B, "Parkes-multibeam-like"): synthetic 8-bit filterbank, 4096
channels, fch1 1518 MHz, foff -0.0703125 MHz, 64 us, 2^20 samples, DM 0-2000 step 2
(1001 trials), boxcar widths 1..4096, baseline 2 s, threshold 6, 2^18-sample
chunks (5 overlapping chunks, overlap = max_delay + boxcar_max), 10 injected
pulses.  One step = the whole file through the hot path: every chunk's
dedispersion + detection chain, the file-level candidate sort and link_grid.

  value : DM-trial*samples/s = ntrials * nsamples * steps / device time, payload
          resident in HBM (4 GiB > L2, so no L2 flush is needed between steps)
  e2e   : the same through the C ABI from pinned host memory: the 4 GiB payload
          H2D (copy stream, overlapped) and the candidate/cluster D2H are inside
          every timed step
  roofline : the dominant kernel (dedispersion) is CUDA-core-ALU bound (~460
          channel-adds per algorithmic byte): achieved channel-adds/s over the
          measured 32-bit add peak of this GPU (pgb_microbench_add_peak)
  cpu_baseline : the reference library (oracle/_ref, compiled from the reference's
          own sources) in parity mode on the host cores, on a bounded sample

`--impl reference` times only the reference CPU implementation (rank 0).
Multi-GPU (torchrun, one rank per GPU): DM trials are sharded across ranks, the
candidate lists are gathered with NCCL and rank 0 clusters them (strong scaling:
the file is fixed, each rank does 1/N of the trials).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG_B = dict(workload="config_B_parkes_like", nchans=4096, fch1=1518.0, foff=-0.0703125,
                tsamp=64e-6, nsamples=1 << 20, dm_lo=0.0, dm_hi=2000.0, dm_step=2.0,
                boxcar_max=4096, detect_thresh=6.0, baseline_s=2.0, nsamps_chunk=1 << 18,
                npulses=10, seed=1001)
METRIC = "DM-trial*samples/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- synthetic data ------------------------------------------------------------------

def _noise_table() -> np.ndarray:
    """u16 random -> N(100, 16^2) quantised round-half-up to u8 (inverse CDF table)."""
    from statistics import NormalDist

    nd = NormalDist(100.0, 16.0)
    u = (np.arange(65536) + 0.5) / 65536.0
    x = np.array([nd.inv_cdf(v) for v in u])
    return np.clip(np.floor(x + 0.5), 0, 255).astype(np.uint8)


def pulse_specs(cfg, plan):
    """(trial, t0, width, snr) of the injected pulses, spread over DM, time and width."""
    rng = np.random.default_rng(cfg["seed"])
    out = []
    n = cfg["npulses"]
    for k in range(n):
        trial = int((k + 0.5) / n * (plan.ntrials - 1))
        width = 1 << int(rng.integers(0, 8))
        snr = float(rng.uniform(12.0, 20.0))
        span = cfg["nsamples"] - int(plan.delays[trial].max()) - width - 1
        t0 = int((k + 0.5) / n * span)
        out.append((trial, t0, width, snr))
    return out


def make_payload(cfg, plan, rows: int | None = None, device: str = "cuda"):
    """[rows][nchans] uint8 torch tensor (default: the whole file) on `device`."""
    import torch

    rows = rows or cfg["nsamples"]
    nch = cfg["nchans"]
    table = torch.from_numpy(_noise_table()).to(device)
    g = torch.Generator(device=device)
    g.manual_seed(cfg["seed"])
    out = torch.empty((rows, nch), dtype=torch.uint8, device=device)
    step = 1 << 14
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        idx = torch.randint(0, 65536, ((r1 - r0) * nch,), generator=g, device=device, dtype=torch.int32)
        out[r0:r1] = table[idx].view(r1 - r0, nch)
    chans = torch.arange(nch, device=device)
    for trial, t0, width, snr in pulse_specs(cfg, plan):
        amp = snr * 16.0 / math.sqrt(nch * width)
        d = torch.from_numpy(plan.delays[trial]).to(device)
        for w in range(width):
            r = t0 + d + w
            keep = r < rows
            rr, cc = r[keep], chans[keep]
            v = out[rr, cc].to(torch.float32) + amp
            out[rr, cc] = torch.clamp(torch.floor(v + 0.5), 0, 255).to(torch.uint8)
    return out


def build_task(cfg):
    from paper_2512_00398_b200.dedisp import FilterbankHeader, LinearSpacing
    from paper_2512_00398_b200.engine import EngineConfig, RfiConfig
    from paper_2512_00398_b200.pipeline import SearchParams, create_task

    hdr = FilterbankHeader(fch1=cfg["fch1"], foff=cfg["foff"], nchans=cfg["nchans"],
                           tsamp=cfg["tsamp"], nsamples=cfg["nsamples"])
    params = SearchParams(dm_lo=cfg["dm_lo"], dm_hi=cfg["dm_hi"], spacing=LinearSpacing(cfg["dm_step"]),
                          engine=EngineConfig(n_workers=1, detect_thresh=cfg["detect_thresh"],
                                              boxcar_max=cfg["boxcar_max"]),
                          baseline_len_s=cfg["baseline_s"], nsamps_chunk=cfg["nsamps_chunk"],
                          rfi=RfiConfig(narrowband=cfg.get("rfi", False), broadband=cfg.get("rfi", False)))
    return create_task(hdr, params)


# ---- clocks ------------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = Path(tempfile.mkstemp(prefix="pg_clocks_", suffix=".csv")[1])

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        self.fh.close()

    def summary(self) -> dict:
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---- CPU reference ------------------------------------------------------------------------

def reference_sample(cfg, plan, task, payload_chunk0: np.ndarray, target_s: float, threads: int):
    """Time the reference run_dm_loop (parity mode) on chunk 0 over a strided trial
    subset sized to ~target_s of CPU work.  Returns (rate, wall_s, sample_desc)."""
    from oracle.pyoracle import Reference

    ref = Reference()
    spec = task.chunks[0]
    L = spec.length
    # ~ channel-adds per second of the reference on `threads` cores
    est_rate = 1.2e9 * threads
    per_trial = L * cfg["nchans"]
    ntr = int(max(4, min(plan.ntrials, target_s * est_rate / per_trial)))
    stride = max(1, plan.ntrials // ntr)
    trials = np.arange(0, plan.ntrials, stride)[:ntr]
    dms, delays = plan.dms[trials], plan.delays[trials]
    ecfg = dict(n_workers=threads, tsamp=cfg["tsamp"], detect_thresh=cfg["detect_thresh"],
                boxcar_max=cfg["boxcar_max"], baseline_window=task.engine.baseline_window)
    cands, skipped, ms = ref.run_dm_loop(payload_chunk0, vars(spec), dms, delays, ecfg, parity=True)
    useful = len(trials) * (spec.valid_end - spec.valid_begin)
    desc = (f"chunk 0 of {cfg['workload']} ({L} samples, valid {spec.valid_end - spec.valid_begin}), "
            f"{len(trials)} of {plan.ntrials} trials (every {stride}th), parity mode, {threads} threads")
    return useful / (ms / 1e3), ms / 1e3, desc


def run_reference_arm(args, cfg, rank: int):
    if rank != 0:
        return
    from paper_2512_00398_b200.dedisp import generate_dm_trials  # noqa: F401  (plan only)

    task = build_task(cfg)
    plan = task.plan
    threads = os.cpu_count() or 1
    chunk0 = make_payload(cfg, plan, rows=task.chunks[0].length, device="cpu").numpy()
    per_step = float(os.environ.get("PG_REF_STEP_S", "8.0"))
    for _ in range(args.warmup):
        reference_sample(cfg, plan, task, chunk0, per_step, threads)
    rates, walls, desc = [], [], ""
    for _ in range(args.steps):
        r, w, desc = reference_sample(cfg, plan, task, chunk0, per_step, threads)
        rates.append(r)
        walls.append(w)
    total_units = sum(r * w for r, w in zip(rates, walls))
    value = total_units / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DM-trial*samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "nchans": cfg["nchans"], "nsamples": cfg["nsamples"],
                   "ntrials": plan.ntrials, "boxcar_max": cfg["boxcar_max"],
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "DM-trial*samples/s", "cores": threads,
                         "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": "DM-trial*samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "x_realtime": value / plan.ntrials * cfg["tsamp"],
    }
    print(json.dumps(line), flush=True)


# ---- our arm ------------------------------------------------------------------------------

def load_ncu_traffic() -> float | None:
    p = ROOT / "profiles" / "ncu_dedisp_summary.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["dram_bytes_per_launch"])
        except (KeyError, ValueError):
            return None
    return None


def run_ours(args, cfg, rank: int, world: int, local_rank: int):
    import torch

    from paper_2512_00398_b200 import _native
    from paper_2512_00398_b200.distributed import DD_TRIAL_BLOCK, gather_candidates, shard_trials, trial_work
    from paper_2512_00398_b200.engine import Engine

    # PG_DIST_BACKEND=gloo + PG_SAME_GPU=1 exercise the multi-rank path on one GPU
    # (functional check only: ranks then share the device and the timing is meaningless)
    backend = os.environ.get("PG_DIST_BACKEND", "nccl")
    if os.environ.get("PG_SAME_GPU"):
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    task = build_task(cfg)
    plan = task.plan
    t0 = time.time()
    payload = make_payload(cfg, plan, device=f"cuda:{local_rank}")
    torch.cuda.synchronize()
    log(f"[rank {rank}] payload {tuple(payload.shape)} generated in {time.time() - t0:.1f}s; "
        f"{len(task.chunks)} chunks, {plan.ntrials} trials, baseline window {task.engine.baseline_window}")
    lo, hi = shard_trials(trial_work(plan, [c.length for c in task.chunks]), world, DD_TRIAL_BLOCK)[rank]
    eng = Engine(local_rank)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local_rank}")
    dev = torch.device("cuda", local_rank)

    def step(src, on_host: bool):
        """One file through the hot path; returns (d2h bytes, dedisp ms, dedisp launches, adds)."""
        cands, clusters, _ = eng.search_file(src, cfg["nsamples"], task.chunks, plan, task.engine,
                                             trial_range=(lo, hi), cluster=(world == 1))
        d2h = cands.nbytes + (clusters.records.nbytes + clusters.members.nbytes if world == 1 else 0)
        if world > 1:
            merged = gather_candidates(cands, device=dev if backend == "nccl" else torch.device("cpu"))
            if rank == 0:
                cl = eng.link_grid(merged, task.engine.radii)
                d2h += cl.records.nbytes + cl.members.nbytes
        ms, nl, adds = eng.last_dedisp_time()
        return d2h, ms, nl, adds

    def timed(src, on_host: bool, steps: int):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = eng.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        d2h = 0
        dd_ms = dd_n = dd_adds = 0
        for _ in range(steps):
            b, ms, nl, adds = step(src, on_host)
            d2h += b
            dd_ms += ms
            dd_n += nl
            dd_adds += adds
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        el = ev0.elapsed_time(ev1)
        if dist:
            t = torch.tensor([el], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el, d2h // steps, eng.launch_count() - launches0, dd_ms, dd_n, dd_adds

    for _ in range(args.warmup):
        step(payload, False)
    with ClockSampler(local_rank) as clk:
        el, _, launches, dd_ms, dd_n, dd_adds = timed(payload, False, args.steps)
    units = plan.ntrials * cfg["nsamples"] * args.steps
    value = units / (el / 1e3)

    # e2e through the C ABI from pinned host memory (H2D + D2H inside every step)
    host = payload.cpu().pin_memory()
    step(host, True)
    e2e_steps = max(1, min(args.steps, 5))
    el_e2e, d2h, _, _, _, _ = timed(host, True, e2e_steps)
    e2e_value = plan.ntrials * cfg["nsamples"] * e2e_steps / (el_e2e / 1e3)

    # roofline of the dominant kernel
    peak = _native_add_peak(local_rank)
    per_launch_ms = dd_ms / max(1, dd_n)
    achieved = (dd_adds / max(1, dd_n)) / (per_launch_ms / 1e3)
    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                chunk0 = payload[: task.chunks[0].length].cpu().numpy()
                threads = os.cpu_count() or 1
                rate, wall, desc = reference_sample(cfg, plan, task, chunk0, args.cpu_seconds, threads)
                cpu = {"value": rate, "unit": "DM-trial*samples/s", "cores": threads,
                       "kind": "reference", "sample": desc, "wall_s": wall}
            except Exception as exc:  # the oracle is optional on a box without oracle/_ref
                log(f"cpu baseline unavailable: {exc}")
        result = {
            "metric": METRIC, "value": value, "unit": "DM-trial*samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32 (u8 SWAR dedispersion), fp64 detection", "data": "synthetic",
            "config": {"workload": cfg["workload"], "nchans": cfg["nchans"],
                       "nsamples": cfg["nsamples"], "ntrials": plan.ntrials,
                       "dm": f"{cfg['dm_lo']}-{cfg['dm_hi']} step {cfg['dm_step']}",
                       "boxcar_max": cfg["boxcar_max"], "baseline_s": cfg["baseline_s"],
                       "nsamps_chunk": cfg["nsamps_chunk"], "chunks": len(task.chunks),
                       "parallelism": f"dm-trial shards x{world}",
                       "l2": "inputs larger than L2 (4 GiB payload, 1 GiB chunks)"},
            "x_realtime": (cfg["nsamples"] * cfg["tsamp"]) / (el / 1e3 / args.steps),
            "e2e": {"value": e2e_value, "unit": "DM-trial*samples/s",
                    "h2d_bytes_per_step": int(cfg["nsamples"] * cfg["nchans"]),
                    "d2h_bytes_per_step": int(d2h),
                    "x_realtime": (cfg["nsamples"] * cfg["tsamp"]) / (el_e2e / 1e3 / e2e_steps)},
            "roofline": {"bound": "alu", "kernel": "dedisp_u8_ring_persist_kernel<8,2,3,8>",
                         "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tadd/s",
                         "frac": achieved / peak, "traffic": load_ncu_traffic(),
                         "per_unit": "nchans channel-adds per (trial, output sample)",
                         "launch_ms": per_launch_ms,
                         "note": "peak = measured CUDA-core 32-bit add rate (pgb_microbench_add_peak); "
                                 "dedispersion moves ~2e-3 B per add, far right of the HBM ridge"},
            "dedisp_share": (dd_ms / args.steps) / (el / args.steps),
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if cpu:
            result["cpu_baseline"] = cpu
        print(json.dumps(result), flush=True)
    eng.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


def _native_add_peak(device: int) -> float:
    import ctypes

    from paper_2512_00398_b200._native import check, lib

    v = ctypes.c_double()
    check(lib.pgb_microbench_add_peak(device, ctypes.byref(v), None))
    return v.value


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="approximate CPU work of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to the contract minimum of 3")
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = dict(CONFIG_B)
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return
    run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
