"""Config E one-chunk file search (ablation library): the product's fp32 path vs the
event-replay kernel (PGB_RFI_HYB=1), interleaved, identical candidates required."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402
from tools import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "E1"
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dict(synth.CONFIGS[name])
task = bench.build_task(cfg)
payload = bench.make_payload(cfg, task.plan)
t = {"f32": [], "hyb": []}
ref = None
with Engine(0, ablations=True) as eng:
    for it in range(trials + 1):
        for mode in ("f32", "hyb"):
            os.environ.pop("PGB_RFI_HYB", None)
            if mode == "hyb":
                os.environ["PGB_RFI_HYB"] = "1"
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c, _, _ = eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if it:
                t[mode].append(el)
            if ref is None:
                ref = c
            else:
                same = len(c) == len(ref) and all(np.array_equal(c[k], ref[k]) for k in ref.dtype.names)
                assert same, (mode, len(c), len(ref))
            print(mode, round(el * 1e3, 1), "ms", eng.last_dedisp_time(), file=sys.stderr, flush=True)
print(json.dumps({"config": name, "f32_ms": [round(1e3 * x, 1) for x in t["f32"]],
                  "hyb_ms": [round(1e3 * x, 1) for x in t["hyb"]], "candidates": int(len(ref)),
                  "identical": True}))
