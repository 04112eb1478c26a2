"""Hint orders, TP groups and the arbitration twin (mirrors rrfp/arbitration.py).

``HintOrder`` (arbitration.py:40-66), ``TpGroup`` (69-82) and ``Decision``
(85-90) keep the reference's names and validation.  ``arbitrate_snapshot``
evaluates one decision through the C-ABI ``rrfp_arbitrate`` -- the same
__host__ __device__ code the device dispatcher and replay kernel run.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

from . import _lib
from .workload import BACKWARD, FORWARD, WEIGHT, TaskId

HINT_KINDS = ("bf", "fb", "bprio", "fprio", "bfw", "external")
NORMAL, DRAIN_BACKWARD, FOCUS_MICROBATCH = "normal", "drain_backward", "focus_microbatch"
_MODE_CODE = {NORMAL: 0, DRAIN_BACKWARD: 1, FOCUS_MICROBATCH: 2}


@dataclass(frozen=True)
class HintOrder:
    kind: str = "bf"
    ranked: tuple = ()

    def __post_init__(self):
        if self.kind not in HINT_KINDS:
            raise ValueError(f"unknown hint kind: {self.kind}")
        if self.kind == "external":
            if not self.ranked:
                raise ValueError("external hint needs a ranked list")
            for d, rule in self.ranked:
                if d not in (FORWARD, BACKWARD, WEIGHT) or rule not in ("asc", "desc"):
                    raise ValueError(f"bad external hint entry: {(d, rule)}")

    @classmethod
    def parse(cls, text: str) -> "HintOrder":
        return cls(kind=text.lower())


@dataclass(frozen=True)
class TpGroup:
    group_size: int = 1
    coordination_round_cost: int = 5
    skew_lo: int = 0
    skew_hi: int = 0

    def __post_init__(self):
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.skew_lo < 0 or self.skew_hi < self.skew_lo:
            raise ValueError("skew bounds must satisfy 0 <= lo <= hi")


class Decision(NamedTuple):
    kind: str
    task: TaskId | None


WAIT = Decision("wait", None)


def _bits(arr, keys, mw):
    for mb, c in keys:
        k = c * mw * 32 + mb
        arr[k >> 5] |= 1 << (k & 31)


def arbitrate_snapshot(*, stage: int, num_microbatches: int, num_chunks: int,
                       decompose: bool, hint: HintOrder, forward_ready=(), backward_ready=(),
                       weight_pending=(), admission=None, mode=NORMAL, focus=-1, phase="",
                       done=()) -> Decision:
    """One arbitration decision via the C twin.  Sets are (mb, chunk) pairs;
    ``done`` holds (mb, chunk, "F"|"B") like ``StageProgress.done``."""
    L = _lib.lib()
    st = _lib.StageState()
    st.M, st.C = num_microbatches, num_chunks
    st.MW = (num_microbatches + 31) // 32
    st.decompose = int(decompose)
    st.admission = -1 if admission is None else admission
    st.mode = _MODE_CODE[mode]
    st.focus = focus
    st.phase = {"": -1, FORWARD: _lib.DIR_F, BACKWARD: _lib.DIR_B}[phase]
    _bits(st.fready, forward_ready, st.MW)
    _bits(st.bready, backward_ready, st.MW)
    _bits(st.wpend, weight_pending, st.MW)
    _bits(st.doneF, [(m, c) for m, c, d in done if d == FORWARD], st.MW)
    _bits(st.doneB, [(m, c) for m, c, d in done if d == BACKWARD], st.MW)
    out = _lib.Decision_()
    _lib.check(L.rrfp_arbitrate(_lib.C.byref(st), _lib.C.byref(_lib.make_hint(hint)),
                                _lib.C.byref(out)))
    if out.kind == _lib.WAIT:
        return WAIT
    d = _lib.CODE_DIR[out.kind]
    return Decision(d, TaskId(stage, out.mb, out.chunk, d))
