"""A/B of the file search's back-half stream (ablation library): back halves on their own
stream (default) vs on the main stream (PGB_BACK_MAIN=1), interleaved trials on config B
(the bench workload) and config A; candidates must be identical.  One JSON line per config."""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from tools import synth  # noqa: E402
from paper_2512_00398_b200.engine import Engine  # noqa: E402


def one(eng, task, payload, cfg):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c, _, _ = eng.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, c


def main():
    names = sys.argv[1:] or ["B", "A"]
    trials = 8
    with Engine(0, ablations=True) as eng:
        for name in names:
            cfg = dict(synth.CONFIGS[name])
            task = bench.build_task(cfg)
            payload = bench.make_payload(cfg, task.plan)
            t = {"side": [], "main": []}
            ref = None
            for mode in ("side", "main"):  # warm-up both
                os.environ.pop("PGB_BACK_MAIN", None)
                if mode == "main":
                    os.environ["PGB_BACK_MAIN"] = "1"
                one(eng, task, payload, cfg)
            for _ in range(trials):
                for mode in ("side", "main"):
                    os.environ.pop("PGB_BACK_MAIN", None)
                    if mode == "main":
                        os.environ["PGB_BACK_MAIN"] = "1"
                    s, c = one(eng, task, payload, cfg)
                    t[mode].append(s)
                    if ref is None:
                        ref = c
                    else:
                        assert len(c) == len(ref) and all(np.array_equal(c[k], ref[k]) for k in ref.dtype.names)
            os.environ.pop("PGB_BACK_MAIN", None)
            print(json.dumps({"config": name, "side_ms_median": 1e3 * float(np.median(t["side"])),
                              "main_ms_median": 1e3 * float(np.median(t["main"])),
                              "side_ms": [round(1e3 * x, 2) for x in t["side"]],
                              "main_ms": [round(1e3 * x, 2) for x in t["main"]],
                              "candidates": int(len(ref)), "identical": True}), flush=True)


if __name__ == "__main__":
    main()
