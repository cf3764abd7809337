"""Per-shard time of the config-B file search on ONE GPU, for world sizes 1/2/4/8: the
work each rank of `bench.py --gpus N` does (its contiguous trial block, whole file),
timed with CUDA events, max over shards.  Predicts the strong-scaling efficiency the
8-GPU run would show before the (tiny) candidate gather; it is not a multi-GPU run.

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
        print(json.dumps({"world": world, "ms_per_step_max_shard": worst,
                          "value": plan.ntrials * cfg["nsamples"] / (worst / 1e3),
                          "efficiency_vs_1": res[1] / (world * worst)}), flush=True)
