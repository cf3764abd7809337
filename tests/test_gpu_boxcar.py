"""The boxcar ladder: the prefix-sum kernel (exact int64
range sums of a tile, src/detect.cpp:211-221 restated where the tree's partial sums are
provably exact) and the reference-order tree kernel it hands the other tiles to."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2512_00398_b200.engine import Chunk, ChunkSpec, EngineConfig
from tests.helpers import assert_same_candidates, cfg_dict, u8_chunk
from tests.test_gpu_parity import _float_workload, _small_u8_case

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _spiky(ref, spikes):
    """The float workload with huge single-sample spikes: a tile holding a spike spans more
    than 2^24 in magnitude, so its range sums are not provably exact -> the tree kernel."""
    hdr, plan, g = _float_workload(ref)
    for t, c, v in spikes:
        g[t, c] = np.float32(v)
    return hdr, plan, g


@pytest.mark.parametrize("window", [0, 1001])
@pytest.mark.parametrize("bmax", [64, 4096])
def test_spike_tiles_match_reference(engine, ref, window, bmax):
    hdr, plan, g = _spiky(ref, [(1000, 3, 3.0e9), (6000, 17, -2.5e9), (7000, 0, 1.0e-30)])
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=bmax, baseline_window=window)
    spec = ChunkSpec.whole(g.shape[0])
    want, want_sk, _ = ref.run_dm_loop(g, vars(spec), plan.dms, plan.delays, cfg_dict(cfg))
    res = engine.run_dm_loop(Chunk(spec, g), plan, cfg)
    assert len(want) > 0
    assert_same_candidates(res.candidates, want)
    assert np.array_equal(res.skipped_trials, want_sk)


@pytest.mark.parametrize("bmax", [1, 2, 16, 256, 2048, 4096, 8192, 16384])
def test_prefix_equals_tree(engine, abl_engine, monkeypatch, bmax):
    """Every ladder geometry (tile of 8192 or 12288 samples, T = N - bmax odd for bmax = 1,
    the register levels, the global levels above 8192): the prefix kernel and the tree
    kernel (PGB_BOXCAR_TREE=1, ablation library) give identical candidates."""
    hdr, plan, data = _small_u8_case()
    L = data.shape[0]
    if L < 3 * bmax:
        data = np.concatenate([data] * (3 * bmax // L + 1))[: 3 * bmax + 5000]
        L = data.shape[0]
    cfg = EngineConfig(n_workers=2, tsamp=hdr.tsamp, boxcar_max=bmax, baseline_window=2001, detect_thresh=4.0)
    spec = ChunkSpec.whole(L)
    a = engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    monkeypatch.setenv("PGB_BOXCAR_TREE", "1")
    b = abl_engine.run_dm_loop(Chunk(spec, data), plan, cfg)
    assert len(a.candidates) > 0
    assert_same_candidates(a.candidates, b.candidates)


SPIKE = """
import sys; sys.path.insert(0, {root!r})
from oracle import pyoracle
from tests.test_gpu_boxcar import _spiky
from paper_2512_00398_b200.engine import Chunk, ChunkSpec, Engine, EngineConfig
hdr, plan, g = _spiky(pyoracle.Reference(), [(1000, 3, 3.0e9)])
with Engine(0) as e:
    e.run_dm_loop(Chunk(ChunkSpec.whole(g.shape[0]), g), plan,
                  EngineConfig(n_workers=1, tsamp=hdr.tsamp, boxcar_max=64, baseline_window=0))
print("ok")
"""


def test_spike_tiles_are_handed_to_the_tree_kernel():
    """PGB_DD_WHICH logs how many tiles the prefix kernel could not prove exact: a spike
    makes some (the trials whose series cross it), not all."""
    if not (ROOT / "oracle" / "_ref").exists():
        pytest.skip("reference library not built")
    e = dict(os.environ, PGB_DD_WHICH="1")
    out = subprocess.run([sys.executable, "-c", SPIKE.format(root=str(ROOT))], env=e, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
    lines = [ln for ln in out.stderr.splitlines() if ln.startswith("pgb boxcar:")]
    assert lines, out.stderr[-2000:]
    nfb, tot = int(lines[-1].split()[4]), int(lines[-1].split()[6])
    assert 0 < nfb < tot, lines

