"""Regenerate the golden fixtures from the compiled reference library.

Run in the dev container (needs oracle/_ref, i.e. /root/reference at build time):
    python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py) and the device path
(tests/test_gpu_parity.py) on machines without the reference sources.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle.pyoracle import Reference  # noqa: E402


def u8_case():
    """128-ch, 12000-sample u8 chunk with three injected pulses (same as the GPU tests)."""
    ref = Reference()
    fch1, foff, tsamp, nch, L = 1500.0, -1.0, 64e-6, 128, 12000
    dms, delays = ref.generate_dm_trials(0.0, 120.0, fch1, foff, tsamp, nch, step=4.0)
    rng = np.random.default_rng(7)
    grid = rng.normal(100.0, 16.0, (L, nch))
    for trial, t0, width, snr in [(15, 3000, 8, 25.0), (22, 7000, 1, 14.0), (5, 9500, 64, 18.0)]:
        amp = snr * 16.0 / np.sqrt(nch * width)
        for c in range(nch):
            s = t0 + int(delays[trial, c])
            grid[s: s + width, c] += amp
    data = np.clip(np.floor(grid + 0.5), 0, 255).astype(np.uint8)
    return dict(fch1=fch1, foff=foff, tsamp=tsamp), dms, delays, data


def main():
    ref = Reference()
    out = {}
    # known answers of the reference tests
    out["delay_426"] = ref.delay_samples(100.0, 1500.0, -1.0, 64e-6, 101, 100)
    _, d501 = ref.generate_dm_trials(0.0, 1000.0, 1500.0, -1.0, 64e-6, 501, step=250.0)
    out["max_delay_36014"] = int(d501.max())
    dad, _ = ref.generate_dm_trials(0.0, 1000.0, 1500.0, -1.0, 64e-6, 64, tol=1.25)
    out["adaptive_count_10328"] = len(dad)
    # config-B plan (all delays): 1001 x 4096 int32 would be 16 MB -> keep a hash + corners
    dmsb, delb = ref.generate_dm_trials(0.0, 2000.0, 1518.0, -0.0703125, 64e-6, 4096, step=2.0)
    out["planB_dms"] = dmsb
    out["planB_delays_sum"] = np.int64(delb.sum())
    out["planB_delays_rows"] = delb[::100].copy()
    # run_dm_loop on the u8 case (parity mode)
    hdr, dms, delays, data = u8_case()
    spec = dict(index=0, start_sample=0, length=data.shape[0], overlap=0, valid_begin=0,
                valid_end=data.shape[0])
    cfg = dict(n_workers=4, tsamp=hdr["tsamp"], detect_thresh=6.0, boxcar_max=256, baseline_window=2001)
    cands, skipped, _ = ref.run_dm_loop(data, spec, dms, delays, cfg)
    out["u8_data"] = data
    out["u8_dms"] = dms
    out["u8_delays"] = delays
    out["u8_cands"] = cands
    out["u8_skipped"] = skipped
    # float engine workload (tests/test_engine.cpp:17-33)
    g = ref.generate_noise(1500.0, -2.0, 64e-6, 32, 8192, 0.0, 1.0, 77)
    ref.inject_pulse(g, 1500.0, -2.0, 64e-6, 100.0, 2000 * 64e-6, 4, ref.amplitude_for_snr(18.0, 1.0, 32, 4))
    ref.inject_pulse(g, 1500.0, -2.0, 64e-6, 40.0, 5000 * 64e-6, 8, ref.amplitude_for_snr(15.0, 1.0, 32, 8))
    fdms, fdel = ref.generate_dm_trials(0.0, 150.0, 1500.0, -2.0, 64e-6, 32, step=2.0)
    fspec = dict(index=0, start_sample=0, length=8192, overlap=0, valid_begin=0, valid_end=8192)
    fcfg = dict(n_workers=2, tsamp=64e-6, detect_thresh=6.0, boxcar_max=64, baseline_window=1001)
    fc, fs, _ = ref.run_dm_loop(g, fspec, fdms, fdel, fcfg)
    out["f32_noise"] = g
    out["f32_dms"] = fdms
    out["f32_delays"] = fdel
    out["f32_cands"] = fc
    out["f32_skipped"] = fs
    # link_grid on the u8 candidates and the .cand text
    clusters, members, _ = ref.link_grid(cands, (3, 9, 3))
    out["u8_clusters"] = clusters
    out["u8_members"] = members
    out["u8_cand_text"] = np.frombuffer(ref.write_candidates(clusters).encode(), np.uint8)
    np.savez_compressed(HERE / "golden_ref.npz", **out)
    print({k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()})


if __name__ == "__main__":
    main()
