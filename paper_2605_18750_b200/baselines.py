"""Fixed-order schedules (mirrors rrfp/baselines.py:34-91).

The schedule is lowered to a per-stage task-code list that the replay
kernel (virtual clock) and the free-running dispatcher (FIXED mode) follow:
the head of the list runs as soon as it is ready, later entries never
overtake it (baselines.py:121-143).
"""

from __future__ import annotations

from dataclasses import dataclass

from .workload import BACKWARD, FORWARD, TaskId, Workload


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
    orders = []
    for s in range(n):
        warm = min(m, n - 1 - s)
        seq = [TaskId(s, j, 0, FORWARD) for j in range(warm)]
        for j in range(m - warm):
            seq.append(TaskId(s, warm + j, 0, FORWARD))
            seq.append(TaskId(s, j, 0, BACKWARD))
        seq += [TaskId(s, j, 0, BACKWARD) for j in range(m - warm, m)]
        orders.append(tuple(seq))
    return FixedSchedule(tuple(orders))
