"""Time the link-substituted reference pipeline (oracle/_ref/pipeline_b200: the reference's
create_task + execute_task with paper_2512_00398_b200/dropin linked in place of
engine.o / cluster.o) on the config-B file, and the pure Python/C-ABI paths beside it.

    python tools/dropin_timing.py [--runs 3]
Prints one JSON line per path (execute_task wall/read/dm_loop/cluster ms as the
reference's FileOutcome reports them) with nvidia-smi clocks."""
import argparse
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from tests.helpers import task_for  # noqa: E402
from tools import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=3)
    args = ap.parse_args()
    cfg = dict(synth.CONFIGS["B"])
    td = Path(tempfile.mkdtemp(prefix="pg_dropin_"))
    fil = td / "B.fil"
    synth.write_filterbank(fil, cfg, task_for(cfg).plan.delays)
    argv = [str(ROOT / "oracle/_ref/pipeline_b200"), str(fil), str(td / "b.cand"), str(cfg["dm_lo"]),
            str(cfg["dm_hi"]), str(cfg["dm_step"]), str(cfg["boxcar_max"]), str(cfg["baseline_s"]),
            str(cfg["nsamps_chunk"]), "16"]
    subprocess.run(argv, check=True, capture_output=True)  # warm-up (page cache, CUDA init)
    units = 1001 * cfg["nsamples"]
    for _ in range(args.runs):
        with bench.ClockSampler(0) as clk:
            t0 = time.perf_counter()
            out = subprocess.run(argv, check=True, capture_output=True, text=True)
            wall = time.perf_counter() - t0
        rec = json.loads(out.stdout)
        rec.update(path="link-substituted reference execute_task (pipeline_b200, process incl. CUDA init)",
                   process_s=wall, value_execute_task=units / (rec["wall_ms"] / 1e3),
                   x_realtime=cfg["nsamples"] * cfg["tsamp"] / (rec["wall_ms"] / 1e3), clocks=clk.summary())
        print(json.dumps(rec), flush=True)
    from paper_2512_00398_b200.pipeline import search_fil
    from tests.test_gpu_stream import _params

    search_fil(fil, _params(cfg))  # warm-up
    for _ in range(args.runs):
        with bench.ClockSampler(0) as clk:
            t0 = time.perf_counter()
            res = search_fil(fil, _params(cfg))
            wall = time.perf_counter() - t0
        print(json.dumps({"path": "pipeline.search_fil (streamed from the .fil, bounded memory)", "wall_ms": 1e3 * wall,
                          "value": units / wall, "x_realtime": cfg["nsamples"] * cfg["tsamp"] / wall,
                          "clusters": len(res.clusters), "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
