"""One config-B chunk through run_dm_loop (device-resident payload): the command the
ncu captures under profiles/ are taken on.  Not a benchmark (no timing)."""
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
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
with Engine(0) as eng:
    for _ in range(reps):
        res = eng.run_dm_loop(Chunk(spec, payload), task.plan, task.engine)
    print(f"chunk 0: {len(res.candidates)} candidates, {len(res.skipped_trials)} skipped; "
          f"dedisp {eng.last_dedisp_time()}")
