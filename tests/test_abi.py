"""The C ABI boundary and the host-side mirror of the reference interface (no GPU needed)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2512_00398_b200 import abi, errors
from paper_2512_00398_b200._native import LIB_PATH, lib
from paper_2512_00398_b200.dedisp import (AdaptiveSpacing, FilterbankHeader, LinearSpacing,
                                          adaptive_dm_step, delay_samples, generate_dm_trials)
from paper_2512_00398_b200.engine import (EngineConfig, in_flight_limit, partition_trials,
                                          trial_working_set_bytes)

from .conftest import HAVE_GPU

HEADER = Path(__file__).resolve().parents[1] / "include" / "pulsegrid_b200.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(pgb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/pulsegrid_b200.h but not exported"
    assert lib.pgb_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_record_layouts():
    # pulsegrid::Candidate is 72 bytes (detect.hpp:14-25); ChunkSpec 48 (filterbank.hpp:48-55)
    assert abi.CANDIDATE_DTYPE.itemsize == 72
    assert abi.CHUNK_SPEC_DTYPE.itemsize == 48
    assert abi.CLUSTER_DTYPE.itemsize == 120


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    from paper_2512_00398_b200.engine import Engine

    with pytest.raises(errors.DeviceError):
        Engine(0)


def test_plan_generation_matches_reference(ref):
    hdr = FilterbankHeader(fch1=1518.0, foff=-0.0703125, nchans=4096, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 2000.0, hdr, LinearSpacing(2.0))
    dms, delays = ref.generate_dm_trials(0.0, 2000.0, 1518.0, -0.0703125, 64e-6, 4096, step=2.0)
    assert np.array_equal(plan.dms, dms) and np.array_equal(plan.delays, delays)
    assert plan.max_delay == 29423
    h64 = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=64, tsamp=64e-6)
    assert adaptive_dm_step(1.25, h64) == ref.adaptive_dm_step(1.25, 1500.0, -1.0, 64e-6, 64)
    assert generate_dm_trials(0.0, 1000.0, h64, AdaptiveSpacing(1.25)).ntrials == 10328
    h101 = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=101, tsamp=64e-6)
    assert delay_samples(100.0, h101, 100) == 426


def test_plan_errors():
    h = FilterbankHeader(fch1=1500.0, foff=-1.0, nchans=8, tsamp=64e-6)
    with pytest.raises(errors.InvalidRangeError):
        generate_dm_trials(10.0, 5.0, h, LinearSpacing(1.0))
    with pytest.raises(errors.InvalidRangeError):
        generate_dm_trials(0.0, 10.0, h, LinearSpacing(0.0))
    with pytest.raises(errors.InvalidRangeError):
        generate_dm_trials(0.0, 10.0, h, AdaptiveSpacing(1.0))


def test_engine_host_arithmetic():
    # tests/test_engine.cpp:52-68 and :130-145
    parts = partition_trials(7, 3)
    assert parts == [[0, 3, 6], [1, 4], [2, 5]]
    h = FilterbankHeader(fch1=1500.0, foff=-2.0, nchans=32, tsamp=64e-6)
    plan = generate_dm_trials(0.0, 150.0, h, LinearSpacing(2.0))
    cfg = EngineConfig(baseline_window=1001)
    ws = trial_working_set_bytes(plan, 8192, cfg)
    cfg.memory_budget = ws
    assert in_flight_limit(plan, 8192, cfg) == 1
    cfg.memory_budget = ws * 10 + ws // 2
    assert in_flight_limit(plan, 8192, cfg) == 10
    cfg.memory_budget = ws - 1
    with pytest.raises(errors.ConfigError):
        in_flight_limit(plan, 8192, cfg)


def test_status_codes_map_to_reference_exceptions():
    assert issubclass(errors.ChunkTooShortError, errors.PulsegridError)
    with pytest.raises(errors.ChunkTooShortError) as ei:
        errors.raise_for(abi.ERR_CHUNK_TOO_SHORT, "trial 7: chunk of 10 samples cannot cover")
    assert ei.value.trial_index == 7
    with pytest.raises(errors.ConfigError):
        errors.raise_for(abi.ERR_CONFIG, "x")
    errors.raise_for(abi.OK, "")


def test_product_library_reads_no_ablation_switches():
    """The alternative kernels and schedules of DESIGN.md section 10 are selected by PGB_*
    environment variables only in libpgb200_ablations.so; the product library references
    just the diagnostics (trace, kernel-choice log) and the initial buffer capacity."""
    import re

    from paper_2512_00398_b200._native import ABLATION_LIB_PATH, LIB_PATH

    names = set(re.findall(rb"PGB_[A-Z0-9_]+", LIB_PATH.read_bytes()))
    assert names <= {b"PGB_TRACE", b"PGB_DD_WHICH", b"PGB_INITIAL_CAP"}, names
    if ABLATION_LIB_PATH.exists():
        abl = set(re.findall(rb"PGB_[A-Z0-9_]+", ABLATION_LIB_PATH.read_bytes()))
        assert {b"PGB_NO_OVERLAP_REUSE", b"PGB_RING_MODE", b"PGB_SYNC_BACK"} <= abl
