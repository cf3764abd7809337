import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from tools import synth
import bench
from paper_2512_00398_b200.engine import Engine
cfg = dict(synth.CONFIGS["E1"])
task = bench.build_task(cfg)
payload = synth.payload(cfg, task.plan.delays)
with Engine(0) as e:
    t = time.time()
    c, cl, sk = e.search_file(payload, cfg["nsamples"], task.chunks, task.plan, task.engine, rfi=task.rfi)
    print("E1", len(c), time.time() - t, file=sys.stderr)
