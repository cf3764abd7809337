"""Config-B file search from a pinned host payload (bench.py's e2e leg), PGB_TRACE=1
timeline of the last of REPS runs.  Not a benchmark.     python tools/trace_e2e.py [reps]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402
from tools import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = dict(bench.CONFIG_B)
task = bench.build_task(cfg)
host_t = torch.empty((cfg["nsamples"], cfg["nchans"]), dtype=torch.uint8, pin_memory=True)
host = host_t.numpy()
synth.payload(cfg, task.plan.delays, out=host)
with Engine(0) as eng:
    for i in range(reps):
        if i == reps - 1:
            os.environ["PGB_TRACE"] = "1"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.search_file(host, cfg["nsamples"], task.chunks, task.plan, task.engine)
        torch.cuda.synchronize()
        print(f"run {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
