"""Config B streamed from a .fil on disk (pipeline.search_fil: parallel preads into two
pinned chunk buffers while the previous chunk computes) at several reader thread counts,
with the reader-wait time the engine records.  python tools/fil_timing.py [threads ...]"""
import json
import os
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
    threads = [int(a) for a in sys.argv[1:]] or [4, 8, 16]
    cfg = dict(synth.CONFIGS["B"])
    td = Path(tempfile.mkdtemp(prefix="pg_fil_"))
    fil = td / "B.fil"
    synth.write_filterbank(fil, cfg, task_for(cfg).plan.delays)
    from paper_2512_00398_b200.engine import default_engine
    from paper_2512_00398_b200.pipeline import search_fil
    from tests.test_gpu_stream import _params

    units = 1001 * cfg["nsamples"]
    search_fil(fil, _params(cfg))  # warm-up (page cache, CUDA init)
    for nt in threads:
        for _ in range(2):
            with bench.ClockSampler(0) as clk:
                t0 = time.perf_counter()
                res = search_fil(fil, _params(cfg), read_threads=nt)
                wall = time.perf_counter() - t0
            st = default_engine(0).last_stream_times()
            print(json.dumps({"path": "pipeline.search_fil", "read_threads": nt, "wall_ms": 1e3 * wall,
                              "value": units / wall, "x_realtime": cfg["nsamples"] * cfg["tsamp"] / wall,
                              "clusters": len(res.clusters), "cpus": os.cpu_count(), **st,
                              "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
