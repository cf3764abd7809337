"""Candidate merging: pulsegrid's cluster.hpp API on the B200.

`link_grid(cands, radii)` is the drop-in for pulsegrid::link_grid
(/root/reference/proj/include/pulsegrid/cluster.hpp:43, src/cluster.cpp:99-146):
identical clusters, representatives, extents and member ids, clusters sorted by
the representative's (peak_sample, dm_trial, width_index).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import abi
from .engine import LinkRadii, default_engine


@dataclass
class Clusters:
    """Flat form of std::vector<ClusterResult> (cluster.hpp:20-28)."""

    records: np.ndarray   # abi.CLUSTER_DTYPE
    members: np.ndarray   # uint64 member ids; cluster k owns members[off : off + count]

    def __len__(self) -> int:
        return len(self.records)

    def member_ids(self, k: int) -> np.ndarray:
        off = int(self.records["member_offset"][k])
        cnt = int(self.records["members"][k])
        return self.members[off: off + cnt]

    @property
    def representatives(self) -> np.ndarray:
        return self.records["representative"]


def linked(a, b, radii: LinkRadii) -> bool:
    """src/cluster.cpp:77-88, for host-side checks."""
    dt = abs(int(a["peak_sample"]) - int(b["peak_sample"]))
    wmax = max(int(a["width_samples"]), int(b["width_samples"]))
    if dt > radii.sep_time * wmax:
        return False
    if abs(int(a["dm_trial"]) - int(b["dm_trial"])) > radii.sep_dm_trials:
        return False
    return abs(int(a["width_index"]) - int(b["width_index"])) <= radii.sep_width


def link_grid(cands: np.ndarray, radii: LinkRadii | None = None, *, device: int = 0) -> Clusters:
    """pulsegrid::link_grid on the device."""
    return default_engine(device).link_grid(np.ascontiguousarray(cands, abi.CANDIDATE_DTYPE), radii)
