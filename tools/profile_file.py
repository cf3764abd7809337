"""Config-B file searches (device-resident payload) for shard RANK of WORLD, for ncu launch
lists and PGB_TRACE=1 timelines (the last of REPS runs is the warm one).  Not a benchmark.
    python tools/profile_file.py [world] [rank] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_00398_b200.distributed import DD_TRIAL_BLOCK, shard_trials, trial_work  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = dict(bench.CONFIG_B)
task = bench.build_task(cfg)
payload = bench.make_payload(cfg, task.plan)
torch.cuda.synchronize()
lo, hi = shard_trials(trial_work(task.plan, [c.length for c in task.chunks]), world, DD_TRIAL_BLOCK)[rank]
with Engine(0) as eng:
    for _ in range(reps - 1):
        eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine,
                        trial_range=(lo, hi), cluster=(world == 1))
    cands, _, _ = eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine,
                                  trial_range=(lo, hi), cluster=(world == 1))
    print(f"shard {rank}/{world}: trials [{lo}, {hi}), {len(cands)} candidates")
