"""A reduced config-E chunk (8192 channels, E's band and DM step, 1024 trials, 2^16 samples,
the E RFI pattern) through the device file search: the command the fp16 kernel's ncu
captures are taken on.  Not a benchmark."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402
from tools import synth  # noqa: E402

cfg = dict(synth.CONFIGS["E"], workload="config_E_profile", nsamples=1 << 16, nsamps_chunk=1 << 16,
           dm_hi=511.5, seed=5002)
task = bench.build_task(cfg)
payload = synth.payload(cfg, task.plan.delays)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
import os
with Engine(0, ablations=bool(os.environ.get("PG_TEST_ABLATIONS"))) as e:
    for _ in range(reps):
        c, cl, sk = e.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)
        print("dedisp", e.last_dedisp_time(), flush=True)
    print(f"{task.plan.ntrials} trials, {len(c)} candidates, dedisp {e.last_dedisp_time()}")
