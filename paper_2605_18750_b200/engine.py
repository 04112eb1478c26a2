"""Replay engine: the reference's virtual-clock scheduler, executed on the B200.

``run_rrfp`` / ``run_fixed`` keep the signatures of rrfp.engine.run_rrfp
(engine.py:452-466) and rrfp.baselines.run_fixed (baselines.py:94-172) and
return the same ``(Trace, Metrics)``.  The tick loop runs as ONE CUDA kernel
(``rrfp_replay_device``, csrc/rrfp_replay.cu): one thread per stage, ready
sets as bitmasks, lock-step ticks.  The dispatch order it produces is the
"replay" schedule the free-running runtime (runtime.py) can then follow with
real compute, and it is bit-exact against the CPU oracle (tests/).

``device="cpu"`` runs the same state machine through the C++ host twin
(``rrfp_replay_host``); it is an explicit choice for CPU-only test runs,
never a silent fallback.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .arbitration import HintOrder, TpGroup
from .jitter import JitterConfig
from .tables import DeviceTables, lower
from .trace import Metrics, StageMetrics, Trace, TraceEvent
from .workload import BACKWARD, FORWARD, Workload


class EngineDeadlockError(RuntimeError):
    def __init__(self, message: str, dump: str = ""):
        super().__init__(message)
        self.dump = dump


def _as_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def replay_tables(tb: DeviceTables, device: str = "cuda"):
    """Run the replay engine on lowered tables; returns (events, ReplayResult)."""
    L = _lib.lib()
    cap = L.rrfp_replay_event_capacity(C.byref(tb.desc))
    if cap <= 0:
        _lib.check(-1)
    res = _lib.ReplayResult()
    if device == "cpu":
        ev = (_lib.Event * cap)()
        rc = L.rrfp_replay_host(C.byref(tb.desc), _as_ptr(tb.dur), _as_ptr(tb.comm),
                                _as_ptr(tb.skew), _as_ptr(tb.fixed), ev, cap, C.byref(res))
        if rc not in (0, -2):
            _lib.check(rc)
        return list(ev[:res.n_events]), res
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("run on the B200: no CUDA device (use device='cpu' for the host twin)")
    dev = torch.device(device)
    ws_bytes = L.rrfp_replay_workspace_bytes(C.byref(tb.desc))
    t_dur = torch.from_numpy(tb.dur.ravel()).to(dev)
    t_comm = torch.from_numpy(tb.comm.ravel()).to(dev)
    t_skew = torch.from_numpy(tb.skew.ravel()).to(dev)
    t_fixed = torch.from_numpy(tb.fixed.ravel().view(np.int32)).to(dev)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    evbuf = torch.empty(cap * C.sizeof(_lib.Event), dtype=torch.uint8, device=dev)
    resbuf = torch.zeros(C.sizeof(_lib.ReplayResult), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(L.rrfp_replay_device(
        C.byref(tb.desc), C.c_void_p(t_dur.data_ptr()), C.c_void_p(t_comm.data_ptr()),
        C.c_void_p(t_skew.data_ptr()), C.c_void_p(t_fixed.data_ptr()),
        C.c_void_p(ws.data_ptr()), C.c_void_p(evbuf.data_ptr()), cap,
        C.c_void_p(resbuf.data_ptr()), C.c_void_p(stream.cuda_stream)))
    stream.synchronize()
    res = _lib.ReplayResult.from_buffer_copy(resbuf.cpu().numpy().tobytes())
    raw = evbuf[: res.n_events * C.sizeof(_lib.Event)].cpu().numpy().tobytes()
    ev = list((_lib.Event * res.n_events).from_buffer_copy(raw)) if res.n_events else []
    return ev, res


def _max_overlap(ivs) -> int:
    marks = sorted([(a, 1) for a, _ in ivs] + [(max(a, b), -1) for a, b in ivs])
    cur = peak = 0
    for _, dlt in marks:
        cur += dlt
        peak = max(peak, cur)
    return peak


def gaps(windows, horizon):
    """Maximal idle intervals in [0, horizon] (engine._gaps semantics)."""
    out, prev, merged = [], 0, []
    for a, b in sorted(windows):
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    for a, b in merged:
        if a > prev:
            out.append((prev, a))
        prev = max(prev, b)
    if prev < horizon:
        out.append((prev, horizon))
    return out


def build_trace_metrics(workload: Workload, ev, res, *, record_trace=True, fixed=False,
                        clock="virtual", time_scale=1.0):
    """Device event records -> (Trace, Metrics) with the reference's fields,
    including occupancy peaks reconstructed from exec/recv/send records
    (engine.py:398-430 interval semantics)."""
    n, r = workload.num_stages, workload.tp_group_size
    makespan = int(res.makespan)
    events = []
    exec_end = {}
    recv_t = {}
    sends = []
    windows = [[] for _ in range(n)]
    for e in ev:
        kind = _lib.EVENT_KINDS[e.kind]
        rank = None if e.rank < 0 else e.rank
        if e.kind == 4:
            d = s = mb = c = None
            stage = e.stage
        else:
            d, stage, mb, c = _lib.task_fields(e.task)
        if e.kind == 0:
            exec_end[(d, stage, mb, c, rank or 0)] = e.t1
            if rank in (None, 0):
                windows[stage].append((e.t0, e.t1))
        elif e.kind == 2:
            recv_t[(d, stage, mb, c, rank)] = e.t0
        elif e.kind == 1:
            sends.append((stage, d, e.t0, e.t1))
        elif e.kind in (3, 4):
            windows[e.stage].append((e.t0, e.t1))
        if record_trace:
            events.append(TraceEvent(int(e.t0), int(e.t1), int(stage), rank, mb, c, d, kind))
    metrics = Metrics(makespan=makespan, total_tasks=workload.task_count(),
                      agreed_rounds=int(res.agreed), deferred_rounds=int(res.deferred))
    nn, cc, m = workload.num_stages, workload.num_chunks, workload.num_microbatches
    for s in range(n):
        occ = {}
        if not fixed:
            for buf in ("forward_ready", "forward_finished", "backward_ready", "backward_finished"):
                worst = 0
                for rank in range(r if buf.endswith("ready") else 1):
                    ivs = []
                    for mb in range(m):
                        for c in range(cc):
                            b_end = exec_end.get((BACKWARD, s, mb, c, rank), makespan)
                            if buf == "forward_ready":
                                t = recv_t.get((FORWARD, s, mb, c, rank))
                                if t is not None:
                                    ivs.append((t, b_end))
                            elif buf == "backward_ready":
                                f_end = exec_end.get((FORWARD, s, mb, c, rank))
                                if s == nn - 1 and c == cc - 1:
                                    t = f_end
                                else:
                                    a = recv_t.get((BACKWARD, s, mb, c, rank))
                                    t = None if a is None or f_end is None else max(a, f_end)
                                if t is not None:
                                    ivs.append((t, b_end))
                    if buf.endswith("finished"):
                        want = FORWARD if buf == "forward_finished" else BACKWARD
                        ivs = [(a, b) for st, d, a, b in sends if st == s and d == want]
                    worst = max(worst, _max_overlap(ivs))
                occ[buf] = worst
        compute, coord = int(res.compute[s]), int(res.coord[s])
        sm = StageMetrics(stage=s, compute=compute, blocking=makespan - compute - coord,
                          tp_coord=coord, n_f=int(res.n_f[s]), n_b=int(res.n_b[s]),
                          n_w=int(res.n_w[s]), max_occupancy=occ)
        metrics.per_stage.append(sm)
        if record_trace:
            for a, b in gaps(windows[s], makespan):
                events.append(TraceEvent(a, b, s, None, None, None, None, "block"))
    return Trace(events=events, clock=clock, time_scale=time_scale), metrics


def run_rrfp(workload: Workload, hint: HintOrder | str = "bf", buffer_limit: int = 32,
             seed: int = 0, *, jitter: JitterConfig | None = None, tp: TpGroup | None = None,
             record_trace: bool = True, device: str = "cuda"):
    """Readiness-driven iteration on the virtual clock (device replay kernel)."""
    if isinstance(hint, str):
        hint = HintOrder.parse(hint)
    tb = lower(workload, hint, buffer_limit, seed, jitter, tp)
    ev, res = replay_tables(tb, device)
    if res.status == -2:
        rem = [int(res.remaining[s]) for s in range(workload.num_stages)]
        raise EngineDeadlockError(
            f"quiescent with {sum(rem)} unfinished tasks", f"remaining per stage: {rem}")
    if res.status != 0:
        _lib.check(res.status)
    return build_trace_metrics(workload, ev, res, record_trace=record_trace)


def run_fixed(schedule, workload: Workload, injected_delays=None, record_trace: bool = True,
              device: str = "cuda"):
    """Fixed-order execution (head blocks; baselines.run_fixed semantics)."""
    from .baselines import ScheduleDeadlockError
    schedule.validate_for(workload)
    tb = lower(workload, HintOrder("bf"), 1 << 30, 0, None, None,
               fixed_order=schedule.per_stage_order, injected=injected_delays or {})
    ev, res = replay_tables(tb, device)
    if res.status == -2:
        raise ScheduleDeadlockError("schedule-induced deadlock")
    if res.status != 0:
        _lib.check(res.status)
    tr, met = build_trace_metrics(workload, [e for e in ev if e.kind == 0], res,
                                  record_trace=record_trace, fixed=True)
    for sm in met.per_stage:
        sm.n_w = 0
    return tr, met
