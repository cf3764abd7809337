"""Dedispersion kernel time for one config-B chunk under the current environment
(variant switches such as PGB_RING_MODE select the ablation library): CUDA-event time of the dedispersion
launch, best of N runs after a warm-up.  Usage: python tools/dd_variant_timing.py [reps]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_00398_b200.engine import Chunk, Engine  # noqa: E402

cfg = dict(bench.CONFIG_B)
task = bench.build_task(cfg)
spec = task.chunks[0]
payload = bench.make_payload(cfg, task.plan, rows=spec.length)
torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
env = {k: v for k, v in os.environ.items() if k.startswith("PGB_")}
with Engine(0, ablations=bool(env)) as eng:
    ts = []
    for _ in range(reps + 1):
        res = eng.run_dm_loop(Chunk(spec, payload), task.plan, task.engine)
        ms, n, adds = eng.last_dedisp_time()
        ts.append(ms)
    best = min(ts[1:])
    print(f"{env} dedisp best {best:.3f} ms  ({adds / best / 1e9:.2f} Tadd/s)  all {[round(t, 2) for t in ts]}  "
          f"cands {len(res.candidates)}")
