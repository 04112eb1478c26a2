"""Lower a Workload (+ jitter, TP group, fixed schedule) to the device tables.

Layout (include/rrfp_b200.h, "replay engine"): per stage, a dense key space
``key = chunk * 32*MW + mb`` so ready sets are chunk-major bitmasks.

* ``dur``  int64[N, 3, KEYS]   latency + injected jitter (dir B=0, F=1, W=2)
* ``comm`` int64[N, 2, KEYS]   delay of the message SENT by (s, dir, key)
* ``skew`` int64[N, 2, KEYS, R] arrival skew of the message TO (s, dir, key) at rank r
* ``fixed`` uint32[N, per_stage] FIXED-mode order (task codes)

Everything random is drawn here on the host with the reference's own
stream derivation (rng.substream), never on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .arbitration import HintOrder, TpGroup
from .jitter import JitterConfig, build_injection_table
from .rng import substream
from .workload import (BACKWARD, FORWARD, WEIGHT, DependencyEdge, TaskId, Workload, route)

DIR_IDX = {BACKWARD: 0, FORWARD: 1, WEIGHT: 2}


@dataclass
class DeviceTables:
    desc: _lib.IterDesc
    dur: np.ndarray
    comm: np.ndarray
    skew: np.ndarray
    fixed: np.ndarray
    injected: dict
    keys: int


def key_of(mb: int, chunk: int, mw: int) -> int:
    return chunk * mw * 32 + mb


def lower(workload: Workload, hint: HintOrder, buffer_limit: int, seed: int,
          jitter: JitterConfig | None = None, tp: TpGroup | None = None,
          fixed_order=None, injected=None) -> DeviceTables:
    if buffer_limit < 1:
        raise ValueError("buffer_limit must be >= 1")
    # fixed schedules are rank-agnostic (baselines.run_fixed runs one lane)
    r = 1 if fixed_order is not None else workload.tp_group_size
    if fixed_order is not None:
        tp = None
    if tp is None:
        tp = TpGroup(group_size=r)
    elif tp.group_size != r:
        raise ValueError("TpGroup.group_size must match workload.tp_group_size")
    n, m, cc = workload.num_stages, workload.num_microbatches, workload.num_chunks
    mw = (m + 31) // 32
    keys = cc * mw * 32
    if injected is None:
        injected = build_injection_table(workload, jitter or JitterConfig(), seed)

    dur = np.zeros((n, 3, keys), np.int64)
    for t, lat in workload.latency.items():
        dur[t.stage, DIR_IDX[t.direction], key_of(t.microbatch, t.chunk, mw)] = \
            lat + injected.get(t, 0)

    comm = np.zeros((n, 2, keys), np.int64)
    skew = np.zeros((n, 2, keys, r), np.int64)
    for s in range(n):
        for mb in range(m):
            for c in range(cc):
                for d in (FORWARD, BACKWARD):
                    src = TaskId(s, mb, c, d)
                    dst = route(workload, src)
                    if dst is None or dst == "turnaround":
                        continue
                    dtask, kind = dst
                    comm[s, DIR_IDX[d], key_of(mb, c, mw)] = \
                        workload.comm_delay.sample(DependencyEdge(src, dtask, kind))
                    if tp.skew_hi > 0 and r > 1:
                        dk = key_of(dtask.microbatch, dtask.chunk, mw)
                        for rank in range(r):
                            rng = substream(seed, "skew", dtask.key(), rank)
                            skew[dtask.stage, DIR_IDX[dtask.direction], dk, rank] = \
                                int(rng.integers(tp.skew_lo, tp.skew_hi + 1))

    per_stage = m * cc * (3 if workload.decompose_backward else 2)
    fixed = np.zeros((n, per_stage), np.uint32)
    if fixed_order is not None:
        for s, order in enumerate(fixed_order):
            if len(order) != per_stage:
                raise ValueError(f"stage {s} order must list exactly its own tasks")
            fixed[s] = [_lib.task_code(t.direction, t.stage, t.microbatch, t.chunk) for t in order]

    d = _lib.IterDesc()
    d.N, d.M, d.C, d.R, d.MW = n, m, cc, r, mw
    d.decompose = int(workload.decompose_backward)
    d.buffer_limit = buffer_limit
    d.fixed_mode = int(fixed_order is not None)
    d.per_stage = per_stage
    d.coord_cost = tp.coordination_round_cost
    d.hint = _lib.make_hint(hint)
    return DeviceTables(d, dur, comm, skew, fixed, injected, keys)
