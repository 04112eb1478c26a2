"""The ready-set arbiter surface of rrfp/arbitration.py, backed by the C twin.

Same names, signatures, field names and error behaviour as the reference
(/root/reference/pkg/src/rrfp/arbitration.py), so code written against the
reference's arbiter (e.g. its own tests/test_arbitration.py) runs unchanged:

* ``HintOrder`` 40-66, ``TpGroup`` 69-82, ``Decision`` / ``WAIT`` 85-90
* ``StageBuffers`` 93-116, ``BackpressureState`` 132-145, ``StageProgress``
  159-185, ``ArbiterState`` 218-229 -- the state containers (plain Python)
* ``next_by_priority`` 119-129, ``update_backpressure`` 188-215,
  ``arbitrate`` 232-303 -- evaluated by the C-ABI ``rrfp_next_by_priority`` /
  ``rrfp_update_backpressure`` / ``rrfp_arbitrate``: the dict/set state is
  lowered to the chunk-major bitmasks the device dispatcher holds, and the
  SAME ``__host__ __device__`` code the dispatcher and the replay kernel run
  (csrc/rrfp_core.cuh) makes the decision
* ``advance_round_phase`` 306-320 and ``tp_coordinate`` 323-334 -- scalar
  rules, restated (the device twins are rrfp_advance_phase / the K4 round).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import NamedTuple

from . import _lib
from .workload import BACKWARD, FORWARD, WEIGHT, TaskId

__all__ = [
    "StageBuffers", "BackpressureState", "HintOrder", "TpGroup", "Decision", "ArbiterState",
    "StageProgress", "next_by_priority", "arbitrate", "advance_round_phase",
    "update_backpressure", "tp_coordinate", "arbitrate_snapshot", "WAIT",
    "NORMAL", "DRAIN_BACKWARD", "FOCUS_MICROBATCH", "HINT_KINDS",
]

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


@dataclass
class StageBuffers:
    """One rank's ready views of a stage (arbitration.py:93-116); entries map
    task -> ready time.  ``admission`` is stage 0's next chunk-0 forward."""

    forward_ready: dict = field(default_factory=dict)
    backward_ready: dict = field(default_factory=dict)
    forward_finished: dict = field(default_factory=dict)
    backward_finished: dict = field(default_factory=dict)
    weight_pending: dict = field(default_factory=dict)
    admission: TaskId | None = None

    def forward_candidates(self) -> list:
        cands = list(self.forward_ready)
        if self.admission is not None:
            cands.append(self.admission)
        return cands

    def backward_candidates(self) -> list:
        return list(self.backward_ready)


@dataclass
class BackpressureState:
    """Forward-lead accounting of one stage (arbitration.py:132-145)."""

    limit: int
    n_f: int = 0
    n_b: int = 0
    mode: str = NORMAL
    focus_microbatch: int = -1
    focus_position: int = 0

    @property
    def lead(self) -> int:
        return self.n_f - self.n_b


def local_completion_order(workload, microbatch: int) -> list:
    """F_0..F_{C-1}, B_{C-1}..B_0 of one microbatch, stage -1 (arbitration.py:148-156)."""
    c = workload.num_chunks
    return ([TaskId(-1, microbatch, k, FORWARD) for k in range(c)]
            + [TaskId(-1, microbatch, k, BACKWARD) for k in reversed(range(c))])


@dataclass
class StageProgress:
    """Finished local F/B steps, (mb, chunk, dir) (arbitration.py:159-185)."""

    num_chunks: int
    done: set = field(default_factory=set)

    def mark(self, task: TaskId) -> None:
        if task.direction != WEIGHT:
            self.done.add((task.microbatch, task.chunk, task.direction))

    def microbatch_finished(self, mb: int) -> bool:
        return all((mb, c, d) in self.done for c in range(self.num_chunks)
                   for d in (FORWARD, BACKWARD))

    def next_in_completion_order(self, mb: int):
        pos = 0
        for c in range(self.num_chunks):
            if (mb, c, FORWARD) not in self.done:
                return pos, TaskId(-1, mb, c, FORWARD)
            pos += 1
        for c in reversed(range(self.num_chunks)):
            if (mb, c, BACKWARD) not in self.done:
                return pos, TaskId(-1, mb, c, BACKWARD)
            pos += 1
        return pos, None


@dataclass
class ArbiterState:
    """Round position of the alternating hints (arbitration.py:218-225)."""

    phase: str = ""

    def reset(self) -> None:
        self.phase = ""


# ------------------------------------------------------------- lowering
_PHASE_CODE = {"": -1, FORWARD: _lib.DIR_F, BACKWARD: _lib.DIR_B}
_CODE_MODE = {v: k for k, v in _MODE_CODE.items()}


def _shape(workload, *task_sets):
    """(M, C, MW) of the bitmask lowering: the workload's shape, widened to
    cover every key the caller put in the buffers."""
    m, c = workload.num_microbatches, workload.num_chunks
    for ts in task_sets:
        for t in ts:
            m = max(m, t.microbatch + 1)
            c = max(c, t.chunk + 1)
    mw = (m + 31) // 32
    if m > 1024 or c > 16 or c * mw > _lib.MAX_WORDS:
        raise ValueError(f"arbiter state too large for the device bitmasks (M={m}, C={c})")
    return m, c, mw


def _state(workload, progress, m, c, mw, decompose, admission=-1):
    st = _lib.StageState()
    st.M, st.C, st.MW, st.decompose, st.admission = m, c, mw, int(decompose), admission
    _bits(st.doneF, [(mb, ch) for mb, ch, d in progress.done if d == FORWARD], mw)
    _bits(st.doneB, [(mb, ch) for mb, ch, d in progress.done if d == BACKWARD], mw)
    return st


def next_by_priority(candidates, direction: str):
    """Highest-priority entry of one direction (arbitration.py:119-129):
    forward min (chunk, mb), otherwise min (-chunk, mb).  Evaluated by the
    device dispatcher's ordered-bitmask scan (rrfp_next_by_priority)."""
    cands = list(candidates)
    if not cands:
        return None
    m = max(t.microbatch for t in cands) + 1
    c = max(t.chunk for t in cands) + 1
    mw = (m + 31) // 32
    if m > 1024 or c > 16 or c * mw > _lib.MAX_WORDS:   # beyond the device key space
        key = (lambda t: (t.chunk, t.microbatch)) if direction == FORWARD else \
              (lambda t: (-t.chunk, t.microbatch))
        return min(cands, key=key)
    words = (_lib.C.c_uint32 * _lib.MAX_WORDS)()
    _bits(words, [(t.microbatch, t.chunk) for t in cands], mw)
    out = _lib.Decision_()
    _lib.check(_lib.lib().rrfp_next_by_priority(words, c, mw, int(direction == FORWARD),
                                                _lib.C.byref(out)))
    return next(t for t in cands if (t.microbatch, t.chunk) == (out.mb, out.chunk))


def update_backpressure(bp: BackpressureState, workload, progress: StageProgress) -> BackpressureState:
    """Backpressure mode before an arbitration round (arbitration.py:188-215),
    through the C twin rrfp_update_backpressure.  Returns ``bp`` itself when
    nothing changes, otherwise an updated copy (the reference's ``replace``)."""
    m, c, mw = _shape(workload, [TaskId(0, mb, ch, d) for mb, ch, d in progress.done])
    st = _state(workload, progress, m, c, mw, workload.decompose_backward)
    st.mode, st.focus = _MODE_CODE[bp.mode], bp.focus_microbatch
    # the reference's interleaved branch scans the workload's microbatches only
    st.M = workload.num_microbatches if c > 1 else m
    _lib.check(_lib.lib().rrfp_update_backpressure(_lib.C.byref(st), bp.limit, bp.n_f, bp.n_b))
    mode, focus = _CODE_MODE[st.mode], st.focus
    pos = progress.next_in_completion_order(focus)[0] if mode == FOCUS_MICROBATCH else 0
    if (mode, focus, pos) == (bp.mode, bp.focus_microbatch, bp.focus_position):
        return bp
    return replace(bp, mode=mode, focus_microbatch=focus, focus_position=pos)


def arbitrate(buffers: StageBuffers, hint: HintOrder, bp: BackpressureState, arb: ArbiterState,
              workload, progress: StageProgress) -> Decision:
    """Select the next task of one stage, or wait (arbitration.py:232-303).

    The buffers are lowered to the dispatcher's bitmasks and the decision is
    made by ``rrfp_arbitrate`` (rrfp_arbitrate_core, the code the device
    lanes run); the returned task is the caller's own TaskId object."""
    fw, bw, ww = list(buffers.forward_ready), list(buffers.backward_ready), list(buffers.weight_pending)
    adm = buffers.admission
    m, c, mw = _shape(workload, fw, bw, ww, [adm] if adm is not None else [],
                      [TaskId(0, mb, ch, d) for mb, ch, d in progress.done],
                      [TaskId(0, bp.focus_microbatch, 0, FORWARD)] if bp.focus_microbatch >= 0 else [])
    if adm is not None and adm.chunk != 0:
        raise ValueError("admission must be a chunk-0 forward (StageBuffers.admission)")
    st = _state(workload, progress, m, c, mw, workload.decompose_backward,
                -1 if adm is None else adm.microbatch)
    st.mode, st.focus, st.phase = _MODE_CODE[bp.mode], bp.focus_microbatch, _PHASE_CODE[arb.phase]
    _bits(st.fready, [(t.microbatch, t.chunk) for t in fw], mw)
    _bits(st.bready, [(t.microbatch, t.chunk) for t in bw], mw)
    _bits(st.wpend, [(t.microbatch, t.chunk) for t in ww], mw)
    out = _lib.Decision_()
    _lib.check(_lib.lib().rrfp_arbitrate(_lib.C.byref(st), _lib.C.byref(_lib.make_hint(hint)),
                                         _lib.C.byref(out)))
    if out.kind == _lib.WAIT:
        return WAIT
    d = _lib.CODE_DIR[out.kind]
    pool = {FORWARD: buffers.forward_candidates(), BACKWARD: bw, WEIGHT: ww}[d]
    task = next(t for t in pool if (t.microbatch, t.chunk) == (out.mb, out.chunk))
    return Decision(d, task)


def advance_round_phase(hint: HintOrder, arb: ArbiterState, decision: Decision) -> None:
    """B hands the next probe to F, F to B; W and waits restart the round
    (arbitration.py:306-320; device twin rrfp_advance_phase)."""
    if hint.kind not in ("bf", "fb", "bfw"):
        return
    if decision.kind == BACKWARD:
        arb.phase = FORWARD
    elif decision.kind == FORWARD:
        arb.phase = BACKWARD
    else:
        arb.reset()


def tp_coordinate(proposals, group: TpGroup):
    """One agreement round (arbitration.py:323-334; device: the K4 round of
    the lanes): agreed iff every rank proposed the same present task."""
    if len(proposals) != group.group_size:
        raise ValueError("one proposal required per rank")
    first = proposals[0]
    if first is not None and all(p == first for p in proposals):
        return ("agreed", first)
    return ("deferred", None)


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
