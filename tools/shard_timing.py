"""Per-shard time of the config-B file search on ONE GPU, for world sizes 1/2/4/8: the
work each rank of `bench.py --gpus N` does (its contiguous trial block, whole file),
timed with CUDA events, max over shards.  Predicts the strong-scaling efficiency the
8-GPU run would show before the (tiny) candidate gather; it is not a multi-GPU run.

The e2e input path of N ranks (PayloadFanout: 1/N of the rows H2D from pinned memory per
rank, the rest pulled from the peers) is timed in parts on this GPU: the pinned H2D of
one rank's slice, and a same-device D2D copy of the (N-1)/N rows it pulls.  NVLink 5 is
not available here, so the pull is also costed at an assumed 700 GB/s per direction
(NVSwitch, one GPU reading seven peers); the prediction takes the slower of the two.

    python tools/shard_timing.py [--steps K]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_00398_b200.distributed import DD_TRIAL_BLOCK, shard_trials, trial_work  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
cfg = dict(bench.CONFIG_B)
task = bench.build_task(cfg)
plan = task.plan
payload = bench.make_payload(cfg, plan)
torch.cuda.synchronize()
work = trial_work(plan, [c.length for c in task.chunks])
res = {}
with Engine(0) as eng:
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
    for world in (1, 2, 4, 8):
        worst = 0.0
        for rank, (lo, hi) in enumerate(shard_trials(work, world, DD_TRIAL_BLOCK)):
            def run():
                return eng.search_file(payload, cfg["nsamples"], task.chunks, plan, task.engine,
                                       trial_range=(lo, hi), cluster=(world == 1))
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                run()
            e1.record(stream)
            torch.cuda.synchronize()
            worst = max(worst, e0.elapsed_time(e1) / args.steps)
        res[world] = worst
        # input path of one rank: pinned H2D of its slice, pull of the rest (D2D proxy)
        nb = cfg["nsamples"] * cfg["nchans"]
        slice_b = nb // world
        host = torch.empty(slice_b, dtype=torch.uint8, pin_memory=True)
        dst = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
        src = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
        def t_copy(fn, reps=5):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        h2d = t_copy(lambda: dst[:slice_b].copy_(host, non_blocking=True))
        pull_b = nb - slice_b
        d2d = t_copy(lambda: dst[slice_b:].copy_(src[slice_b:])) if pull_b else 0.0
        nvl = pull_b / 700e9 * 1e3
        e2e = h2d + max(d2d, nvl) + worst
        print(json.dumps({"world": world, "ms_per_step_max_shard": worst,
                          "value": plan.ntrials * cfg["nsamples"] / (worst / 1e3),
                          "efficiency_vs_1": res[1] / (world * worst),
                          "h2d_slice_ms": h2d, "pull_bytes": pull_b, "pull_d2d_same_gpu_ms": d2d,
                          "pull_nvlink_700GBps_ms": nvl, "e2e_pred_ms": e2e,
                          "e2e_pred_value": plan.ntrials * cfg["nsamples"] / (e2e / 1e3)}), flush=True)
        del host, dst, src
