"""Free-running device runtime: ``run_gpu`` replaces ``rrfp.live.run_live``.

``run_gpu`` keeps run_live's signature (live.py:507-523) and returns the same
``(Trace, Metrics)`` with ``clock="wall"``.  Instead of 3 Python threads per
(stage, rank) over in-process queues, every (stage, rank) is a *lane*: one
CUDA graph per iteration whose dispatcher, bodies and sends all run on the
GPU (csrc/rrfp_exec.cu).  Lanes of one process may sit on one device (tests,
single-GPU replay) or on several; multi-process wiring (one stage per GPU
under torchrun) exchanges inbox addresses as CUDA IPC handles
(``LaneGroup.connect_ipc``).

Modes
  free    lanes arbitrate on what physically arrived (the reference's live path)
  fixed   lanes follow a per-stage order list, head blocking (1F1B baseline)
  replay  the replay kernel (engine.py) computes the virtual-clock dispatch
          order first; lanes then execute exactly that order on the device
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .arbitration import HintOrder, TpGroup
from .baselines import FixedSchedule, build_1f1b_schedule
from .engine import gaps, replay_tables
from .jitter import JitterConfig
from .tables import DIR_IDX, key_of, lower
from .trace import Metrics, StageMetrics, Trace, TraceEvent
from .workload import BACKWARD, FORWARD, WEIGHT, TaskId, Workload


class LiveWatchdogError(RuntimeError):
    def __init__(self, message: str, dump: str = ""):
        super().__init__(message)
        self.dump = dump


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def replay_order(workload: Workload, hint: HintOrder, buffer_limit: int, seed: int,
                 jitter, tp, device="cuda"):
    """Per-stage dispatch order of the virtual-clock engine (device kernel)."""
    tb = lower(workload, hint, buffer_limit, seed, jitter, tp)
    ev, res = replay_tables(tb, device)
    if res.status != 0:
        _lib.check(res.status)
    per = [[] for _ in range(workload.num_stages)]
    for e in ev:
        if e.kind == 0 and e.rank <= 0:
            d, s, mb, c = _lib.task_fields(e.task)
            per[s].append((e.t0, TaskId(s, mb, c, d)))
    return [tuple(t for _, t in sorted(p, key=lambda x: x[0])) for p in per]


class LaneGroup:
    """All lanes of one process.  ``placement[stage][rank]`` -> CUDA ordinal;
    ``local`` lists the (stage, rank) lanes this process owns (default: all)."""

    def __init__(self, workload: Workload, hint: HintOrder | str = "bf", buffer_limit: int = 32,
                 time_scale: float = 1.0, *, seed: int = 0, jitter: JitterConfig | None = None,
                 tp: TpGroup | None = None, mode: str = "free", schedule: FixedSchedule | None = None,
                 placement=None, local=None, bodies=None, compute_kind: int = 0,
                 trace_cap: int | None = None, pad_table_us=None, defer_bodies: bool = False,
                 floor_table_us=None, lane_streams=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("run_gpu needs a CUDA device (B200)")
        if isinstance(hint, str):
            hint = HintOrder.parse(hint)
        if time_scale <= 0:
            raise ValueError("time_scale must be positive")
        if mode not in ("free", "fixed", "replay"):
            raise ValueError(f"unknown mode {mode}")
        self.w, self.hint, self.mode, self.scale = workload, hint, mode, time_scale
        n, r = workload.num_stages, workload.tp_group_size
        self.n, self.r = n, r
        order = None
        if mode == "fixed":
            schedule = schedule or build_1f1b_schedule(workload)
            schedule.validate_for(workload)
            order = schedule.per_stage_order
        elif mode == "replay":
            order = replay_order(workload, hint, buffer_limit, seed, jitter, tp)
        tb = lower(workload, hint, buffer_limit, seed, jitter, tp)
        self.tables = tb
        self._seed, self._jitter, self._tp = seed, jitter, tp
        self.compute_kind = compute_kind
        self.injected = tb.injected
        placement = placement or [[0] * r for _ in range(n)]
        self.local = local or [(s, k) for s in range(n) for k in range(r)]
        keys = tb.keys
        mw = tb.desc.MW
        per_stage = tb.desc.per_stage
        tpg = tp or TpGroup(group_size=r)
        cap = trace_cap or (16 * workload.num_microbatches * workload.num_chunks * (r + 2) + 256)
        self.L = _lib.lib()
        self.lanes = {}
        self.streams = {}
        self._tables = {}
        for (s, k) in self.local:
            d = _lib.LaneDesc()
            d.N, d.M, d.C, d.R, d.MW = n, workload.num_microbatches, workload.num_chunks, r, mw
            d.decompose = int(workload.decompose_backward)
            d.buffer_limit = buffer_limit
            d.fixed_mode = int(order is not None)
            d.per_stage = per_stage
            d.stage, d.rank = s, k
            d.device = placement[s][k]
            d.compute_kind = compute_kind
            d.trace_cap = cap
            d.time_scale = time_scale
            d.coord_cost_ns = int(round(tpg.coordination_round_cost * 1000 * time_scale))
            d.hint = _lib.make_hint(hint)
            h = C.c_void_p()
            _lib.check(self.L.rrfp_runtime_create(C.byref(d), C.byref(h)))
            self.lanes[(s, k)] = h
            dev = torch.device("cuda", placement[s][k])
            # (lane_streams: e.g. a green-context partition's stream, see pipeline.py)
            self.streams[(s, k)] = (lane_streams or {}).get((s, k)) or torch.cuda.Stream(dev)
            # tables (ns)
            if compute_kind == 0:
                dur = tb.dur[s].astype(np.float64) * 1000.0 * time_scale
            else:   # real bodies: the table only carries the jitter pad (K11)
                dur = np.zeros((3, keys))
                for t, v in self.injected.items():
                    if t.stage == s:
                        dur[DIR_IDX[t.direction], key_of(t.microbatch, t.chunk, mw)] = v
                if pad_table_us is not None:
                    dur += pad_table_us[s]
                dur = dur * 1000.0 * time_scale
            dur = np.ascontiguousarray(np.rint(dur).astype(np.int64))
            comm = np.ascontiguousarray(np.rint(tb.comm[s] * 1000.0 * time_scale).astype(np.int64))
            f_dst = s + 1 if s + 1 < n else 0
            b_dst = s - 1 if s > 0 else n - 1
            dskew = np.zeros((2, keys, r), np.int64)
            dskew[DIR_IDX[FORWARD]] = tb.skew[f_dst, DIR_IDX[FORWARD]]
            dskew[DIR_IDX[BACKWARD]] = tb.skew[b_dst, DIR_IDX[BACKWARD]]
            dskew = np.ascontiguousarray(np.rint(dskew * 1000.0 * time_scale).astype(np.int64))
            fixed = np.zeros(max(per_stage, 1), np.uint32)
            if order is not None:
                fixed[:] = [_lib.task_code(t.direction, t.stage, t.microbatch, t.chunk)
                            for t in order[s]]
            floor = None
            if floor_table_us is not None:
                floor = self._floor_ns(floor_table_us[s], keys, time_scale)
            self._tables[(s, k)] = (dur, comm, dskew, fixed, floor)
            _lib.check(self.L.rrfp_runtime_load_tables(h, _ptr(dur), _ptr(comm), _ptr(dskew),
                                                      _ptr(fixed), _ptr(floor) if floor is not None
                                                      else None))
            if bodies is not None:
                arr = bodies[(s, k)]          # 3*M*C raw cudaGraph_t handles (kind*M*C + chunk*M + mb)
                carr = (C.c_void_p * len(arr))(*[C.c_void_p(x or 0) for x in arr])
                _lib.check(self.L.rrfp_runtime_set_bodies(h, carr, len(arr)))
        self.cap = cap
        self.epoch = 0
        if len(self.local) == n * r and not defer_bodies:
            self.connect_local()

    @staticmethod
    def _floor_ns(table_us, keys, scale):
        """[3, KEYS] µs floor table -> contiguous int64 ns; the C side copies
        exactly 3*KEYS entries, so the shape is checked here."""
        a = np.asarray(table_us, np.float64)
        if a.shape != (3, keys):
            raise ValueError(f"floor table must be [3, {keys}] (dir x key), got {a.shape}")
        return np.ascontiguousarray(np.rint(a * 1000.0 * scale).astype(np.int64))

    def set_floor_us(self, floor_by_stage):
        """Replace the lognormal-jitter floor tables (µs, [3, KEYS] per stage)
        between iterations."""
        for (s, k), h in self.lanes.items():
            dur, comm, dskew, fixed, _ = self._tables[(s, k)]
            floor = self._floor_ns(floor_by_stage[s], self.tables.keys, self.scale)
            self._tables[(s, k)] = (dur, comm, dskew, fixed, floor)
            _lib.check(self.L.rrfp_runtime_load_tables(h, _ptr(dur), _ptr(comm), _ptr(dskew),
                                                      _ptr(fixed), _ptr(floor)))

    def set_comm_delay(self, comm_delay):
        """Replace the per-edge communication delays (e.g. a lognormal CommDelay
        of another sigma, config 5) between iterations: the edge table is
        re-lowered exactly as at construction (workload.py:109-117 draws)."""
        from dataclasses import replace
        w = replace(self.w, comm_delay=comm_delay)
        tb = lower(w, self.hint, self.tables.desc.buffer_limit, self._seed, self._jitter, self._tp)
        for (s, k), h in self.lanes.items():
            dur, _, dskew, fixed, floor = self._tables[(s, k)]
            comm = np.ascontiguousarray(np.rint(tb.comm[s] * 1000.0 * self.scale).astype(np.int64))
            self._tables[(s, k)] = (dur, comm, dskew, fixed, floor)
            _lib.check(self.L.rrfp_runtime_load_tables(h, _ptr(dur), _ptr(comm), _ptr(dskew), _ptr(fixed),
                                                      _ptr(floor) if floor is not None else None))
        self.w = w

    def set_latency(self, latency: dict):
        """Replace the workload's nominal per-task latencies (e.g. the measured
        task times of the real bodies) and re-derive the J-preset jitter pads
        from them (jitter.py:97-118: the injected delay scales with the
        observed latency EMA), between iterations.  Real-body lanes only."""
        from dataclasses import replace
        if self.compute_kind != 1:
            raise ValueError("set_latency is for lanes running real task bodies")
        w = replace(self.w, latency=dict(latency))
        tb = lower(w, self.hint, self.tables.desc.buffer_limit, self._seed, self._jitter, self._tp)
        self.injected = tb.injected
        mw = tb.desc.MW
        for (s, k), h in self.lanes.items():
            _, comm, dskew, fixed, floor = self._tables[(s, k)]
            dur = np.zeros((3, tb.keys))
            for t, v in self.injected.items():
                if t.stage == s:
                    dur[DIR_IDX[t.direction], key_of(t.microbatch, t.chunk, mw)] = v
            dur = np.ascontiguousarray(np.rint(dur * 1000.0 * self.scale).astype(np.int64))
            self._tables[(s, k)] = (dur, comm, dskew, fixed, floor)
            _lib.check(self.L.rrfp_runtime_load_tables(h, _ptr(dur), _ptr(comm), _ptr(dskew), _ptr(fixed),
                                                      _ptr(floor) if floor is not None else None))
        self.w = w

    def set_bodies(self, bodies: dict):
        for lane, arr in bodies.items():
            carr = (C.c_void_p * len(arr))(*[C.c_void_p(x or 0) for x in arr])
            _lib.check(self.L.rrfp_runtime_set_bodies(self.lanes[lane], carr, len(arr)))

    def inbox(self, lane):
        p = C.c_void_p()
        _lib.check(self.L.rrfp_runtime_inbox(self.lanes[lane], C.byref(p), None))
        return p.value

    def task_ptr(self, lane):
        p = C.c_void_p()
        _lib.check(self.L.rrfp_runtime_task_ptr(self.lanes[lane], C.byref(p)))
        return p.value

    def connect(self, inboxes: dict):
        """Wire every local lane given the inbox address of every lane."""
        n, r = self.n, self.r
        all_lanes = [inboxes[(s, k)] for s in range(n) for k in range(r)]
        for (s, k), h in self.lanes.items():
            f_dst = s + 1 if s + 1 < n else 0
            b_dst = s - 1 if s > 0 else n - 1
            fw = (C.c_void_p * r)(*[inboxes[(f_dst, q)] for q in range(r)])
            bw = (C.c_void_p * r)(*[inboxes[(b_dst, q)] for q in range(r)])
            peers = (C.c_void_p * (r + n * r))(*([inboxes[(s, q)] for q in range(r)] + all_lanes))
            _lib.check(self.L.rrfp_runtime_connect(h, fw, bw, peers))

    def connect_local(self):
        self.connect({lane: self.inbox(lane) for lane in self.lanes})

    def ipc_handles(self) -> dict:
        out = {}
        for lane, h in self.lanes.items():
            buf = (C.c_char * 64)()
            _lib.check(self.L.rrfp_runtime_inbox_ipc(h, buf))
            out[lane] = bytes(buf)
        return out

    def connect_ipc(self, handles: dict):
        """Multi-process wiring: ``handles`` maps every lane to its 64-byte IPC
        handle (gathered with torch.distributed); local lanes use plain pointers."""
        inboxes = {}
        self._opened = getattr(self, "_opened", [])
        for lane, hd in handles.items():
            if lane in self.lanes:
                inboxes[lane] = self.inbox(lane)
            else:
                p = C.c_void_p()
                _lib.check(self.L.rrfp_ipc_open(hd, C.byref(p)))
                self._opened.append(p.value)
                inboxes[lane] = p.value
        self.connect(inboxes)

    def prepare(self):
        """Instantiate + upload every local lane graph while nothing runs."""
        for lane, h in self.lanes.items():
            _lib.check(self.L.rrfp_runtime_prepare(h, C.c_void_p(self.streams[lane].cuda_stream)))
        self.prepared = True

    def launch(self):
        import torch
        if not getattr(self, "prepared", False):
            self.prepare()
        self.epoch += 1
        for lane, h in self.lanes.items():
            st = self.streams[lane]
            st.wait_stream(torch.cuda.current_stream(st.device))
            _lib.check(self.L.rrfp_runtime_launch(h, self.epoch,
                                                  C.c_void_p(self.streams[lane].cuda_stream)))

    def wait(self, watchdog_secs: float = 30.0):
        """Block until every local lane finished; returns raw events and t0s."""
        out, t0s, failures = [], [], []
        for lane, h in self.lanes.items():
            ev = (_lib.Event * self.cap)()
            n_ev = C.c_int32()
            t0 = C.c_int64()
            rc = self.L.rrfp_runtime_wait(h, C.c_double(watchdog_secs), ev, self.cap,
                                          C.byref(n_ev), C.byref(t0))
            if rc == -3:
                failures.append(self.L.rrfp_last_error().decode())
            elif rc != 0:
                _lib.check(rc)
            out.extend(ev[: n_ev.value])
            t0s.append(t0.value)
        if failures:
            dump = []
            for lane, h in self.lanes.items():
                buf = C.create_string_buffer(512)
                self.L.rrfp_runtime_status(h, buf, 512)
                dump.append(buf.value.decode())
            raise LiveWatchdogError("device runtime watchdog fired: " + "; ".join(failures),
                                    "\n".join(dump))
        return out, t0s

    def run_iteration(self, watchdog_secs: float = 30.0):
        self.launch()
        return self.wait(watchdog_secs)

    def close(self):
        for h in self.lanes.values():
            self.L.rrfp_runtime_destroy(h)
        self.lanes = {}
        for ptr in getattr(self, "_opened", []):   # peer inboxes mapped by connect_ipc
            self.L.rrfp_ipc_close(C.c_void_p(ptr))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def wall_trace(workload: Workload, events, t0_ns: int, time_scale: float = 1.0):
    """Raw lane records (globaltimer ns) -> (Trace, Metrics), live._finalize style."""
    n = workload.num_stages
    evs = []
    for e in events:
        kind = _lib.EVENT_KINDS[e.kind]
        rank = None if e.rank < 0 else e.rank
        if e.kind == 4:
            d = mb = c = None
        else:
            d, _, mb, c = _lib.task_fields(e.task)
        a = (e.t0 - t0_ns) // 1000
        b = (e.t1 - t0_ns) // 1000
        evs.append(TraceEvent(int(a), int(b), int(e.stage), rank, mb, c, d, kind))
    evs.sort(key=lambda e: (e.t_start, e.t_end, e.stage, e.event_kind))
    makespan = max((e.t_end for e in evs if e.event_kind == "exec"), default=0)
    met = Metrics(makespan=makespan, total_tasks=workload.task_count())
    final = list(evs)
    for s in range(n):
        lane = [(e.t_start, e.t_end) for e in evs if e.stage == s and
                e.event_kind in ("exec", "coord") and (e.rank is None or e.rank == 0)]
        mine = [e for e in evs if e.stage == s and e.event_kind == "exec" and (e.rank in (None, 0))]
        compute = sum(e.t_end - e.t_start for e in mine)
        coord = sum(e.t_end - e.t_start for e in evs if e.stage == s and e.event_kind == "coord")
        met.per_stage.append(StageMetrics(
            stage=s, compute=compute, tp_coord=coord, blocking=makespan - compute - coord,
            n_f=sum(e.direction == FORWARD for e in mine),
            n_b=sum(e.direction == BACKWARD for e in mine),
            n_w=sum(e.direction == WEIGHT for e in mine)))
        for a, b in gaps(lane, makespan):
            final.append(TraceEvent(a, b, s, None, None, None, None, "block"))
    met.agreed_rounds = sum(1 for e in evs if e.event_kind == "coord" and e.direction is not None)
    met.deferred_rounds = sum(1 for e in evs if e.event_kind == "coord" and e.direction is None)
    return Trace(events=final, clock="wall", time_scale=time_scale), met


def dispatch_latency(trace, n_stages: int) -> dict:
    """The device dispatcher's cost per decision, read off a wall trace (SURVEY
    8d: "the dispatcher is latency-bound, report ns per decision").

    For consecutive tasks of one (stage, rank) lane: if the second was already
    ready when the first ended (its message had arrived, its F / B had run),
    the gap between them is pure dispatch cost -- completion kernel, the WHILE
    iteration, arbitration, the SWITCH into the next body; otherwise the
    arrival -> start delay is the dispatcher's reaction time to a flag.
    Returns p50 / p90 in microseconds and the sample counts."""
    rk = lambda e: 0 if e.rank is None else e.rank     # (TP=1 execs carry rank None, recvs 0)
    execs = [e for e in trace.events if e.event_kind == "exec"]
    recv = {(e.stage, rk(e), e.microbatch, e.chunk, e.direction): e.t_start
            for e in trace.events if e.event_kind == "recv"}
    end = {(e.stage, rk(e), e.microbatch, e.chunk, e.direction): e.t_end for e in execs}
    lanes = {}
    for e in execs:
        lanes.setdefault((e.stage, rk(e)), []).append(e)
    gaps, react = [], []
    for (s, r), lst in lanes.items():
        lst.sort(key=lambda e: e.t_start)
        for a, b in zip(lst, lst[1:]):
            key = lambda d: (s, r, b.microbatch, b.chunk, d)
            if b.direction == "W":
                ready = end.get(key("B"), 0)
            elif b.direction == "B" and key("B") not in recv:   # last (virtual) stage: its own F
                ready = end.get(key("F"), 0)
            else:
                ready = recv.get(key(b.direction), 0)           # (stage-0 F: always ready)
            (gaps if ready <= a.t_end else react).append(
                b.t_start - (a.t_end if ready <= a.t_end else ready))

    def q(x):
        if not x:
            return None
        x = sorted(x)
        return {"p50": x[len(x) // 2], "p90": x[int(0.9 * (len(x) - 1))], "n": len(x)}
    return {"back_to_back_gap_us": q(gaps), "arrival_to_start_us": q(react)}


def run_gpu(workload: Workload, hint: HintOrder | str = "bf", buffer_limit: int = 32,
            time_scale: float = 1.0, *, seed: int = 0, jitter: JitterConfig | None = None,
            tp: TpGroup | None = None, watchdog_secs: float = 30.0, mode: str = "free",
            schedule: FixedSchedule | None = None, placement=None):
    """One iteration on device lanes with synthetic (latency-table) compute.

    Drop-in for ``run_live``: same arguments plus ``mode`` / ``schedule`` /
    ``placement``.  Raises LiveWatchdogError (with a per-lane dump) if no
    lane finishes within ``watchdog_secs``.
    """
    g = LaneGroup(workload, hint, buffer_limit, time_scale, seed=seed, jitter=jitter, tp=tp,
                  mode=mode, schedule=schedule, placement=placement)
    try:
        events, t0s = g.run_iteration(watchdog_secs)
    finally:
        g.close()
    return wall_trace(workload, events, min(t0s), time_scale)
