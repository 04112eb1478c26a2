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
  replay  every lane makes its own decisions (the same device arbiter + K4
          round as free mode) at the reference engine's VIRTUAL times: a
          message carries its virtual arrival time, each lane publishes a
          lower bound on the virtual time of its future sends, and a lane
          decides at tick T only once every in-neighbour's bound exceeds T
          (conservative PDES; csrc/rrfp_exec.cu "replay").  Nothing is taken
          from the oracle: the resulting trace (virtual times) is compared
          with run_rrfp's event for event by the tests.  With ``schedule``:
          FIXED heads under the same virtual clock (run_fixed semantics).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .arbitration import HintOrder, TpGroup
from .baselines import FixedSchedule, build_1f1b_schedule
from .engine import EngineDeadlockError, build_trace_metrics, gaps, replay_tables
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
                 floor_table_us=None, lane_streams=None, declog_cap: int = 0):
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
        if mode == "fixed" or (mode == "replay" and schedule is not None):
            schedule = schedule or build_1f1b_schedule(workload)
            schedule.validate_for(workload)
            order = schedule.per_stage_order
        self.virtual = mode == "replay"
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
        if self.virtual:   # deferred TP rounds: at most one per arrival tick
            cap += 4 * workload.num_microbatches * workload.num_chunks * r
        self.declog_cap = declog_cap
        vh = self._virtual_bounds(tb, tpg) if self.virtual else None
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
            self._fixed_order = order is not None
            d.per_stage = per_stage
            d.stage, d.rank = s, k
            d.device = placement[s][k]
            d.compute_kind = compute_kind
            d.trace_cap = cap
            d.time_scale = time_scale
            d.coord_cost_ns = int(round(tpg.coordination_round_cost * 1000 * time_scale))
            d.hint = _lib.make_hint(hint)
            d.declog_cap = declog_cap
            if self.virtual:
                d.virtual_clock = 1
                d.coord_cost_ns = int(tpg.coordination_round_cost)       # integer us
                d.v_dmin, d.v_la, d.v_horizon = vh["dmin"][s], vh["la"][(s, k)], vh["horizon"]
            h = C.c_void_p()
            _lib.check(self.L.rrfp_runtime_create(C.byref(d), C.byref(h)))
            self.lanes[(s, k)] = h
            dev = torch.device("cuda", placement[s][k])
            # (lane_streams: e.g. a green-context partition's stream, see pipeline.py)
            self.streams[(s, k)] = (lane_streams or {}).get((s, k)) or torch.cuda.Stream(dev)
            # tables (ns; replay mode: integer virtual us, latency + injected)
            if self.virtual:
                dur = tb.dur[s].astype(np.float64)
            elif compute_kind == 0:
                dur = tb.dur[s].astype(np.float64) * 1000.0 * time_scale
            else:   # real bodies: the table only carries the jitter pad (K11)
                dur = np.zeros((3, keys))
                for t, v in self.injected.items():
                    if t.stage == s:
                        dur[DIR_IDX[t.direction], key_of(t.microbatch, t.chunk, mw)] = v
                if pad_table_us is not None:
                    dur += pad_table_us[s]
                dur = dur * 1000.0 * time_scale
            unit = 1.0 if self.virtual else 1000.0 * time_scale
            dur = np.ascontiguousarray(np.rint(dur).astype(np.int64))
            comm = np.ascontiguousarray(np.rint(tb.comm[s] * unit).astype(np.int64))
            f_dst = s + 1 if s + 1 < n else 0
            b_dst = s - 1 if s > 0 else n - 1
            dskew = np.zeros((2, keys, r), np.int64)
            dskew[DIR_IDX[FORWARD]] = tb.skew[f_dst, DIR_IDX[FORWARD]]
            dskew[DIR_IDX[BACKWARD]] = tb.skew[b_dst, DIR_IDX[BACKWARD]]
            dskew = np.ascontiguousarray(np.rint(dskew * unit).astype(np.int64))
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
    def _virtual_bounds(tb, tpg):
        """Replay-mode constants per lane: the stage's smallest task duration
        (v_dmin), the smallest comm delay + arrival skew of the lane's sends
        (v_la) -- together the PDES lookahead -- and an upper bound of the
        makespan (every instant of a live run has a task, a message or a TP
        round in progress), past which a quiescent lane reports a deadlock."""
        d = tb.desc
        n, m, cc, r, mw = d.N, d.M, d.C, d.R, d.MW
        keys = [key_of(mb, c, mw) for c in range(cc) for mb in range(m)]
        dirs = (0, 1, 2) if d.decompose else (0, 1)
        dmin = [int(min(tb.dur[s, di, k] for di in dirs for k in keys)) for s in range(n)]
        la = {}
        for s in range(n):
            f_dst = s + 1 if s + 1 < n else 0
            b_dst = s - 1 if s > 0 else n - 1
            for q in range(r):
                best = None
                for c in range(cc):
                    # (direction row, destination stage, destination chunk) of the
                    # sends of chunk c (engine._send routing, engine.py:181-209)
                    sends = []
                    if s + 1 < n or c + 1 < cc:
                        sends.append((DIR_IDX[FORWARD], f_dst, c if s + 1 < n else c + 1))
                    if s > 0 or c > 0:
                        sends.append((DIR_IDX[BACKWARD], b_dst, c if s > 0 else c - 1))
                    for di, dst, dc in sends:
                        for mb in range(m):
                            v = int(tb.comm[s, di, key_of(mb, c, mw)] + tb.skew[dst, di, key_of(mb, dc, mw), q])
                            best = v if best is None else min(best, v)
                la[(s, q)] = best or 0
        n_msgs = 2 * n * m * cc
        horizon = (int(tb.dur.sum()) + int(tb.comm.sum()) + int(tb.skew.max(initial=0)) * n_msgs
                   + int(tpg.coordination_round_cost) * (n * d.per_stage + n_msgs * r + n) + 16)
        return {"dmin": dmin, "la": la, "horizon": horizon}

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

    def set_jitter(self, jitter: JitterConfig | None):
        """Switch the J-preset injection table (jitter.py:97-118) between
        iterations, keeping the current latencies (real-body lanes)."""
        self._jitter = jitter
        self.set_latency(self.w.latency)

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
        out, t0s, failures, deadlocks = [], [], [], []
        for lane, h in self.lanes.items():
            ev = (_lib.Event * self.cap)()
            n_ev = C.c_int32()
            t0 = C.c_int64()
            rc = self.L.rrfp_runtime_wait(h, C.c_double(watchdog_secs), ev, self.cap,
                                          C.byref(n_ev), C.byref(t0))
            if rc == -3:
                failures.append(self.L.rrfp_last_error().decode())
            elif rc == -2:
                deadlocks.append(self.L.rrfp_last_error().decode())
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
        if deadlocks:     # replay mode: the virtual clock quiesced (engine.py:363-367)
            raise EngineDeadlockError("quiescent with unfinished tasks", "\n".join(deadlocks))
        return out, t0s

    def decisions(self):
        """The last iteration's decision log of every local lane (declog_cap > 0):
        a list of dicts with the exact inputs of update_backpressure + arbitrate
        and the decision the device made (include/rrfp_b200.h rrfp_runtime_declog)."""
        out = []
        for lane, h in self.lanes.items():
            n, stride = C.c_int32(), C.c_int32()
            _lib.check(self.L.rrfp_runtime_declog(h, None, 0, C.byref(n), C.byref(stride)))
            if n.value == 0:
                continue
            buf = np.zeros(n.value * stride.value, np.uint32)
            _lib.check(self.L.rrfp_runtime_declog(h, buf.ctypes.data_as(C.c_void_p), buf.size,
                                                  C.byref(n), C.byref(stride)))
            for rec in buf.reshape(n.value, stride.value):
                out.append(parse_decision(rec, self.tables.desc.MW))
        return out

    def enable_profile(self, cap: int = 4096):
        """Record every lane_step_kernel run of the following iterations
        (include/rrfp_b200.h rrfp_runtime_profile); cap = 0 disables."""
        for h in self.lanes.values():
            _lib.check(self.L.rrfp_runtime_profile(h, cap))
        self._prof_cap = cap

    def profile(self):
        """{lane: uint64[n, 4]} of the last iteration: step-kernel entry, completion
        done, decision made (ns), kind << 32 | view polls."""
        out = {}
        cap = getattr(self, "_prof_cap", 0)
        for lane, h in self.lanes.items():
            buf = np.zeros((max(cap, 1), 4), np.uint64)
            n = C.c_int32()
            _lib.check(self.L.rrfp_runtime_profile_read(h, buf.ctypes.data_as(C.c_void_p), cap, C.byref(n)))
            out[lane] = buf[:n.value].copy()
        return out

    def make_trace(self, events, t0s):
        """(Trace, Metrics) of one iteration: virtual-clock (replay mode) or wall."""
        if self.virtual:
            return virtual_trace(self.w, events, fixed=self._fixed_order)
        return wall_trace(self.w, events, min(t0s), self.scale)


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


def _i32(x):
    x = int(x)
    return x - (1 << 32) if x >= 1 << 31 else x


def parse_decision(rec, mw):
    """One rrfp_runtime_declog record -> dict of (mb, chunk) sets and scalars."""
    nw = int(rec[13])

    def keys(words):
        out = set()
        for w, v in enumerate(words):
            v = int(v)
            while v:
                b = (v & -v).bit_length() - 1
                k = w * 32 + b
                out.add((k % (mw * 32), k // (mw * 32)))
                v &= v - 1
        return out
    base = 16
    blk = [rec[base + i * nw: base + (i + 1) * nw] for i in range(5)]
    modes = {0: "normal", 1: "drain", 2: "focus"}
    kind = {0: "B", 1: "F", 2: "W", 3: "wait"}[int(rec[10])]
    return {"stage": int(rec[0]), "rank": int(rec[1]), "n_f": int(rec[2]), "n_b": int(rec[3]),
            "mode_in": modes[int(rec[4])], "focus_in": _i32(rec[5]),
            "mode": modes[int(rec[6])], "focus": _i32(rec[7]),
            "phase": {-1: "", 0: "B", 1: "F"}[_i32(rec[8])], "admission": _i32(rec[9]),
            "kind": kind, "task": None if kind == "wait" else (_i32(rec[11]), _i32(rec[12])),
            "t": int(rec[14]) | (int(rec[15]) << 32),
            "fready": keys(blk[0]), "bready": keys(blk[1]), "wpend": keys(blk[2]),
            "doneF": keys(blk[3]), "doneB": keys(blk[4])}


def virtual_trace(workload: Workload, events, fixed: bool = False):
    """Replay-mode lane records (virtual us) -> (Trace, Metrics) exactly as
    engine.run_rrfp / baselines.run_fixed build them (engine.py:381-449):
    compute / coord per stage, agreed / deferred rounds, occupancy peaks
    (through engine.build_trace_metrics), block gaps."""
    from types import SimpleNamespace
    n = workload.num_stages
    comp, coord = [0] * n, [0] * n
    nf, nb, nw = [0] * n, [0] * n, [0] * n
    agreed = deferred = 0
    makespan = 0
    for e in events:
        if e.kind == 0:
            makespan = max(makespan, e.t1)
            if e.rank <= 0:
                d, st, _, _ = _lib.task_fields(e.task)
                comp[st] += e.t1 - e.t0
                if d == FORWARD:
                    nf[st] += 1
                elif d == BACKWARD:
                    nb[st] += 1
                else:
                    nw[st] += 1
        elif e.kind in (3, 4):
            coord[e.stage] += e.t1 - e.t0
            agreed += e.kind == 3
            deferred += e.kind == 4
    res = SimpleNamespace(makespan=makespan, agreed=agreed, deferred=deferred, compute=comp,
                          coord=coord, n_f=nf, n_b=nb, n_w=nw)
    evs = [e for e in events if e.kind == 0] if fixed else list(events)
    tr, met = build_trace_metrics(workload, evs, res, fixed=fixed)
    if fixed:
        for sm in met.per_stage:
            sm.n_w = 0
    return tr, met


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


def dispatcher_profile(records: dict, body_us: float | None = None) -> dict:
    """Summary of LaneGroup.profile() records (device %globaltimer stamps inside
    lane_step_kernel, ns): per decision the completion half (end stamp, jitter
    pad, flag sends), the dispatch half when the next task was already ready
    (one view poll: ballot + arbitrate + SWITCH select), and the time from one
    decision to the next step kernel's entry (the SWITCH-launched body, then
    the WHILE node relaunching the step kernel; minus body_us when the bodies
    have a known length).  Microseconds, p50 / p90."""
    comp, dec_ready, between = [], [], []
    waited = 0
    for recs in records.values():
        if len(recs) == 0:
            continue
        r = recs[recs[:, 0].argsort()].astype(np.int64)
        comp += list((r[:, 1] - r[:, 0]) / 1e3)
        polls = r[:, 3] & 0xFFFFFFFF
        kind = r[:, 3] >> 32
        for i in range(len(r)):
            if polls[i] == 1:
                dec_ready.append((r[i, 2] - r[i, 1]) / 1e3)
            else:
                waited += 1
            if i + 1 < len(r) and kind[i] in (0, 1, 2):    # a body ran between the two step kernels
                between.append((r[i + 1, 0] - r[i, 2]) / 1e3 - (body_us or 0.0))

    def q(x):
        if not x:
            return None
        x = sorted(x)
        return {"p50": round(x[len(x) // 2], 2), "p90": round(x[int(0.9 * (len(x) - 1))], 2), "n": len(x)}
    return {"complete_us": q(comp), "decide_when_ready_us": q(dec_ready), "decisions_that_waited": waited,
            ("graph_relaunch_us" if body_us is not None else "decision_to_next_step_us"): q(between)}


def run_gpu(workload: Workload, hint: HintOrder | str = "bf", buffer_limit: int = 32,
            time_scale: float = 1.0, *, seed: int = 0, jitter: JitterConfig | None = None,
            tp: TpGroup | None = None, watchdog_secs: float = 30.0, mode: str = "free",
            schedule: FixedSchedule | None = None, placement=None, declog: list | None = None,
            declog_cap: int | None = None):
    """One iteration on device lanes with synthetic (latency-table) compute.

    Drop-in for ``run_live``: same arguments plus ``mode`` / ``schedule`` /
    ``placement``.  Raises LiveWatchdogError (with a per-lane dump) if no
    lane finishes within ``watchdog_secs``; in replay mode a virtual-clock
    deadlock raises EngineDeadlockError like run_rrfp.  ``declog`` (a list)
    receives every arbitration the lanes evaluated (LaneGroup.decisions).
    mode="replay" returns the virtual-clock trace (clock "virtual").
    """
    if declog_cap is None:
        declog_cap = (8 * workload.task_count() // workload.num_stages + 64) if declog is not None else 0
    g = LaneGroup(workload, hint, buffer_limit, time_scale, seed=seed, jitter=jitter, tp=tp,
                  mode=mode, schedule=schedule, placement=placement, declog_cap=declog_cap)
    try:
        events, t0s = g.run_iteration(watchdog_secs)
        if declog is not None:
            declog.extend(g.decisions())
        return g.make_trace(events, t0s)
    finally:
        g.close()
