"""Transit-parallel schedule export (transit_parallel.py:37-101 API mirror).

The engines build this schedule on device every step (radix sort of the
step's (transit, pair) keys, run-length groups, three work classes).  These
functions expose the same construction for inspection and parity tests:
``transit_schedule`` returns the raw arrays from ``nd_transit_schedule``;
``build_transit_map`` / ``partition_work_classes`` wrap them in the
reference's TransitGroup / TransitSchedule shapes.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

SMALL_MAX_WORK = 32     # transit_parallel.py:37
LARGE_MIN_WORK = 1024   # transit_parallel.py:38
SUBGROUP_THREADS = 32   # transit_parallel.py:39


def subgroup_size(m_i: int) -> int:
    """Members of one group processed as one contiguous unit (:42-44)."""
    return max(1, SUBGROUP_THREADS // m_i)


@dataclass
class TransitGroup:
    transit: int
    members: np.ndarray
    work: int = 0


@dataclass
class TransitSchedule:
    step: int
    small: list = field(default_factory=list)
    medium: list = field(default_factory=list)
    large: list = field(default_factory=list)
    scheduling_index: dict = field(default_factory=dict)

    def all_groups(self):
        return self.small + self.medium + self.large

    def class_counts(self):
        return len(self.small), len(self.medium), len(self.large)


def transit_schedule(pair_transit, m: int = 1) -> dict:
    """Device export: order (members, group-major), group_start[G+1],
    group_transit[G], group_class[G], sched_index[G]."""
    torch = _lib.require_cuda()
    pt = torch.as_tensor(np.asarray(pair_transit, dtype=np.int64) if not hasattr(pair_transit, "is_cuda")
                         else pair_transit, dtype=torch.int64, device="cuda").contiguous()
    n = pt.numel()
    order = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    gs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    gt = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    gc = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    si = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    G = C.c_int64()
    _lib.check(_lib.load().nd_transit_schedule(_lib.ptr(pt), n, int(m), _lib.ptr(order), _lib.ptr(gs),
                                               _lib.ptr(gt), _lib.ptr(gc), _lib.ptr(si), C.byref(G),
                                               _lib.stream_ptr()), "nd_transit_schedule")
    g = G.value
    return dict(order=order[:n].cpu().numpy(), group_start=gs[:g + 1].cpu().numpy(),
                group_transit=gt[:g].cpu().numpy(), group_class=gc[:g].cpu().numpy(),
                sched_index=si[:g].cpu().numpy())


def build_transit_map(pair_transit) -> list:
    """Groups of pair ids by transit, ascending transit, members sample-major."""
    r = transit_schedule(pair_transit, 1)
    gs = r["group_start"]
    return [TransitGroup(int(t), r["order"][gs[i]:gs[i + 1]])
            for i, t in enumerate(r["group_transit"])]


def partition_work_classes(groups, m_i: int, step: int = 0) -> TransitSchedule:
    """Classes by work = members * m_i with dense per-class ranks (:86-101)."""
    sched = TransitSchedule(step=step)
    for g in groups:
        g.work = len(g.members) * m_i
        cls = sched.small if g.work < SMALL_MAX_WORK else (
            sched.medium if g.work <= LARGE_MIN_WORK else sched.large)
        sched.scheduling_index[g.transit] = len(cls)
        cls.append(g)
    return sched
