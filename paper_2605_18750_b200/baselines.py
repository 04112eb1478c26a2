"""Fixed-order schedules (mirrors rrfp/baselines.py:34-91).

The schedule is lowered to a per-stage task-code list that the replay
kernel (virtual clock) and the free-running dispatcher (FIXED mode) follow:
the head of the list runs as soon as it is ready, later entries never
overtake it (baselines.py:121-143).
"""

from __future__ import annotations

from dataclasses import dataclass

from .workload import BACKWARD, FORWARD, WEIGHT, TaskId, Workload


class ScheduleDeadlockError(RuntimeError):
    def __init__(self, message: str, cycle=()):
        super().__init__(message)
        self.cycle = list(cycle)


@dataclass(frozen=True)
class FixedSchedule:
    per_stage_order: tuple

    def to_json(self) -> dict:
        return {"per_stage_order": [[t.key() for t in st] for st in self.per_stage_order]}

    @classmethod
    def from_json(cls, obj: dict) -> "FixedSchedule":
        return cls(tuple(tuple(TaskId.from_key(k) for k in st) for st in obj["per_stage_order"]))

    def validate_for(self, workload: Workload) -> None:
        if len(self.per_stage_order) != workload.num_stages:
            raise ValueError("schedule stage count mismatch")
        mine = {}
        for t in workload.compute_tasks():
            mine.setdefault(t.stage, set()).add(t)
        for s, order in enumerate(self.per_stage_order):
            if len(order) != len(mine[s]) or set(order) != mine[s]:
                raise ValueError(f"stage {s} order must list exactly its own tasks")


def build_1f1b_schedule(workload: Workload) -> FixedSchedule:
    """Warm-up min(M, N-1-i) forwards, strict F/B alternation, then drain."""
    if workload.num_chunks != 1:
        raise ValueError("1F1B baseline covers non-interleaved workloads only")
    if workload.decompose_backward:
        raise ValueError("1F1B baseline does not decompose backward")
    n, m = workload.num_stages, workload.num_microbatches
    return FixedSchedule(tuple(tuple(build_1f1b_schedule_skeleton(n, m, s)) for s in range(n)))


def build_zb_h1_schedule(workload: Workload) -> FixedSchedule:
    """Zero-bubble-H1-like fixed order for a decomposed (B-input / W) workload
    ("fixed-schedule FIXED mode for arbitrary FixedSchedule
    JSON, e.g. ZB-like"): 1F1B's F/B skeleton, with stage i deferring each
    weight-gradient task W(j) until after B(j + N-1-i), so the W tasks fill the
    cool-down bubbles; the remaining W tasks drain at the end."""
    if workload.num_chunks != 1:
        raise ValueError("ZB-H1 schedule covers non-interleaved workloads only")
    if not workload.decompose_backward:
        raise ValueError("ZB-H1 schedule needs a decomposed backward (W tasks)")
    n, m = workload.num_stages, workload.num_microbatches
    orders = []
    for s in range(n):
        lag = n - 1 - s
        seq, next_w = [], 0
        for t in build_1f1b_schedule_skeleton(n, m, s):
            seq.append(t)
            if t.direction == BACKWARD and t.microbatch - lag >= next_w:
                seq.append(TaskId(s, next_w, 0, WEIGHT))
                next_w += 1
        seq += [TaskId(s, j, 0, WEIGHT) for j in range(next_w, m)]
        orders.append(tuple(seq))
    return FixedSchedule(tuple(orders))


def build_1f1b_schedule_skeleton(n: int, m: int, s: int):
    """Stage s's 1F1B F/B order (warm-up min(m, n-1-s) F, alternate, drain)."""
    warm = min(m, n - 1 - s)
    seq = [TaskId(s, j, 0, FORWARD) for j in range(warm)]
    for j in range(m - warm):
        seq += [TaskId(s, warm + j, 0, FORWARD), TaskId(s, j, 0, BACKWARD)]
    return seq + [TaskId(s, j, 0, BACKWARD) for j in range(m - warm, m)]
