"""Readiness-driven pipeline training iteration of the synthetic GPT on device lanes.

``GpuPipeline`` ties the pieces together for one process:
  * one ``StageCompute`` per local stage (model.py) -- weights, grads, slots,
    mailboxes; neighbours' mailboxes are wired so the last kernel of a task
    writes its payload straight into the receiver's slot;
  * one CUDA graph per (kind, microbatch) per stage, captured once;
  * one device lane per stage (runtime.LaneGroup, compute_kind=1) whose
    dispatcher arbitrates (mode "free"), follows 1F1B ("fixed") or follows
    the replayed virtual-clock order ("replay") and launches the captured
    bodies through a SWITCH node.

``step()`` = one training iteration (all M microbatches: F, B and, with the
BFW hint, W) -> mean loss; the host launches ONE graph per lane per step.
"""

from __future__ import annotations

import torch

from .arbitration import HintOrder, TpGroup
from .jitter import JitterConfig
from .model import GPTConfig, RawBuffer, StageCompute
from .runtime import LaneGroup, wall_trace
from .workload import BACKWARD, FORWARD, WEIGHT, TaskId, Workload


def nominal_workload(cfg: GPTConfig, n_stages: int, n_mb: int, decompose: bool,
                     f_us=None, b_us=None, w_us=None, tp_size: int = 1, n_chunks: int = 1) -> Workload:
    """A Workload describing the GPT iteration (latencies = nominal per-task µs).

    Only the structure matters to the free-running lanes (real kernels set
    the durations); the latency values feed the jitter EMA and the
    replay-mode virtual clock.
    """
    lat = {}
    for s in range(n_stages):
        for c in range(n_chunks):
            for mb in range(n_mb):
                lat[TaskId(s, mb, c, FORWARD)] = int(f_us[s] if f_us else 1000)
                lat[TaskId(s, mb, c, BACKWARD)] = int(b_us[s] if b_us else 2000)
                if decompose:
                    lat[TaskId(s, mb, c, WEIGHT)] = int(w_us[s] if w_us else 1000)
    return Workload(num_stages=n_stages, num_microbatches=n_mb, num_chunks=n_chunks, tp_group_size=tp_size,
                    latency=lat, decompose_backward=decompose)


def lognormal_floor_tables(n_stages, n_mb, nominal_us, sigma, seed, stages=None, n_chunks=1):
    """Per-task duration floors (µs) for injected lognormal compute jitter
    (SURVEY.md 8d, config 5): X ~ LogNormal(0, sigma) drawn on the host per
    (stage, mb, chunk, direction) from the (seed, "cjitter", ...) stream; the
    device pads the task until start + nominal * X.  W shares B's draw so a
    decomposed (BFW) and a fused (1F1B / BF) backward see the same
    perturbation.  Returns {stage: float64[3, KEYS]} (dir rows B=0, F=1, W=2)
    indexed like every lane table, KEYS = C * 32*MW, key = chunk * 32*MW + mb
    (tables.key_of)."""
    import numpy as np
    from .rng import substream
    from .tables import key_of
    mw = (n_mb + 31) // 32
    keys = n_chunks * mw * 32
    out = {}
    for s in (stages if stages is not None else range(n_stages)):
        t = np.zeros((3, keys))
        if sigma > 0:
            for c in range(n_chunks):
                for mb in range(n_mb):
                    k = key_of(mb, c, mw)
                    for d, row in (("F", 1), ("B", 0)):
                        labels = (s, mb, d) if n_chunks == 1 else (s, mb, c, d)
                        x = float(np.exp(substream(seed, "cjitter", *labels).normal(0.0, sigma)))
                        t[row, k] = nominal_us[s][d] * x
                        if d == "B" and nominal_us[s].get("W"):
                            t[2, k] = nominal_us[s]["W"] * x
        out[s] = t
    return out


def measured_nominal(trace, n_stages):
    """Mean per-stage task durations (µs) by direction from a wall trace."""
    out = []
    for s in range(n_stages):
        row = {}
        for d in ("F", "B", "W"):
            xs = [e.t_end - e.t_start for e in trace.execs() if e.stage == s and e.direction == d]
            row[d] = sum(xs) / len(xs) if xs else 0.0
        out.append(row)
    return out


class GpuPipeline:
    """All stages (and, with ``tp_size`` > 1, all TP ranks of every stage) in
    this process.  With ``n_chunks`` = C > 1 (interleaved virtual stages,
    workload.py:251-256) the model is split over V = N*C virtual stages and
    virtual stage v = c*N + s is chunk c of lane s: its F output feeds v+1,
    i.e. (s+1, c) or, from the last stage, the wrap edge (0, c+1).
    ``grid[v][r]`` is virtual stage v, TP rank r; ``stages[v]`` its rank 0.
    TP ranks of a stage share its device; each is its own lane."""

    def __init__(self, cfg: GPTConfig, n_stages: int, n_mb: int, *, hint="bf", buffer_limit=32,
                 mode="free", decompose=None, jitter: JitterConfig | None = None, seed: int = 0,
                 devices=None, stage_latency_us=None, model_seed: int = 1234, data_seed: int = 0,
                 schedule=None, comm_delay=None, tp_size: int = 1, tp: TpGroup | None = None,
                 n_chunks: int = 1, mm=None, head_cost: float = 0.0, gemm_sm_cap: int = 0, w_split: str = "fc",
                 green: bool = False, split: str = "layer", declog_cap: int = 0):
        if mm is not None and (tp_size > 1 or n_chunks > 1):
            raise ValueError("the multimodal pipeline (config 4) runs with TP=1, C=1")
        if isinstance(hint, str):
            hint = HintOrder.parse(hint)
        if decompose is None:
            decompose = hint.kind == "bfw"
        R, C, N = tp_size, n_chunks, n_stages
        V = N * C
        self.cfg, self.N, self.M, self.hint, self.R, self.C = cfg, N, n_mb, hint, R, C
        devices = devices or [0] * N
        f_us, b_us, w_us = stage_latency_us or (None, None, None)
        w = nominal_workload(cfg, N, n_mb, decompose, f_us, b_us, w_us, tp_size=R, n_chunks=C)
        if comm_delay is not None:
            w = Workload(num_stages=w.num_stages, num_microbatches=w.num_microbatches,
                         num_chunks=C, tp_group_size=R, latency=w.latency, comm_delay=comm_delay,
                         decompose_backward=decompose)
        self.workload = w
        if len(set(devices)) > 1:   # one process, several GPUs: neighbours store into each other
            from . import _lib
            for a in set(devices):
                for b in set(devices):
                    if a != b:
                        _lib.check(_lib.lib().rrfp_enable_peer_access(a, b))
        self.comms = {}
        if R > 1:   # one TP group per lane (its virtual stages run one task at a time)
            from .tp import TpComm
            for s in range(N):
                self.comms[s] = [TpComm(r, R, (cfg.seq, cfg.d_model), torch.device("cuda", devices[s]))
                                 for r in range(R)]
                TpComm.connect_local(self.comms[s])
        self.mm = mm
        stage_cfg = (lambda v: mm.vit if v < mm.vit_stages else mm.llm) if mm else (lambda v: cfg)
        self.grid = [[StageCompute(stage_cfg(v), v, V, n_mb, torch.device("cuda", devices[v % N]),
                                   decompose=decompose, seed=model_seed, data_seed=data_seed,
                                   tp_rank=r, tp_size=R, tp=self.comms[v % N][r] if R > 1 else None,
                                   mm=mm, head_cost=head_cost if C == 1 else 0.0, w_split=w_split,
                                   split=split)
                      for r in range(R)] for v in range(V)]
        self.stages = [row[0] for row in self.grid]
        # green=True (single-GPU pipeline emulation): every lane gets a disjoint SM
        # partition (CUDA green context); its bodies are captured on the partition's
        # streams, so their kernels run only there -- an idle stage's SMs stay idle
        self.green_streams = {}
        if green:
            import ctypes
            from . import _lib
            if len(set(devices)) != 1 or R != 1:
                raise ValueError("green partitions emulate a pipeline on ONE device without TP")
            arr = (ctypes.c_void_p * (2 * N))()
            self._green_raw = arr
            sms = ctypes.c_int()
            n_sm = torch.cuda.get_device_properties(devices[0]).multi_processor_count
            _lib.check(_lib.lib().rrfp_green_streams(devices[0], N, max(2, (n_sm // N) & ~1), arr,
                                                     ctypes.byref(sms)))
            self.green_sms = sms.value
            gemm_sm_cap = sms.value & ~1
            for s_ in range(N):
                self.green_streams[s_] = (torch.cuda.ExternalStream(arr[2 * s_], device=devices[0]),
                                          torch.cuda.ExternalStream(arr[2 * s_ + 1], device=devices[0]))
            for v in range(V):
                self.grid[v][0].side = self.green_streams[v % N][1]
        for row in self.grid:
            for st in row:
                st.gemm_sm_cap = gemm_sm_cap
        for v in range(V):
            for r in range(R):
                nxt = self.grid[v + 1] if v + 1 < V else None
                prv = self.grid[v - 1] if v > 0 else None
                self.grid[v][r].connect_outputs(
                    fwd_out=[[q.fwd_in[mb] for q in nxt] for mb in range(n_mb)] if nxt else None,
                    bwd_out=[[q.bwd_in[mb] for q in prv] for mb in range(n_mb)] if prv else None)
        # warm-up: every body once with rank-local all-reduces (every kernel
        # module loaded before any rank spins on a peer), then capture
        kinds = ("F", "B", "W") if decompose else ("F", "B")
        for comms in self.comms.values():
            for c in comms:
                c.local_only = True
        streams = {(v, r): (self.green_streams[v % N][0] if green else
                            torch.cuda.Stream(torch.device("cuda", devices[v % N])))
                   for v in range(V) for r in range(R)}
        # the warm-up streams must see the parameter / token initialisation queued on the
        # current stream: an embedding reading a token buffer that is still being written
        # (with a recycled allocation's bytes in it) indexes out of bounds
        for stream in streams.values():
            stream.wait_stream(torch.cuda.current_stream(stream.device))
        for mb in range(n_mb):
            for kind in kinds:
                for (v, r), stream in streams.items():
                    st = self.grid[v][r]
                    st._cap_stream = stream
                    with torch.cuda.stream(stream):
                        st.run_task(kind, mb)
        for stream in streams.values():
            stream.synchronize()
        for comms in self.comms.values():
            for c in comms:
                c.local_only = False
        raw_v = {(v, r): self.grid[v][r].capture() for v in range(V) for r in range(R)}
        bodies = {}
        for s in range(N):
            for r in range(R):
                arr = [None] * (3 * n_mb * C)
                for c in range(C):
                    raw = raw_v[(c * N + s, r)]
                    for ki in range(3):
                        for mb in range(n_mb):
                            arr[ki * n_mb * C + c * n_mb + mb] = raw[ki * n_mb + mb]
                bodies[(s, r)] = arr
        self.group = LaneGroup(w, hint, buffer_limit, 1.0, seed=seed, jitter=jitter, mode=mode,
                               tp=tp or (TpGroup(group_size=R) if R > 1 else None),
                               placement=[[d] * R for d in devices], bodies=bodies, compute_kind=1,
                               schedule=schedule, declog_cap=declog_cap,
                               lane_streams={(s_, 0): self.green_streams[s_][0] for s_ in self.green_streams})
        self.last_events = None

    def step(self, watchdog_secs: float = 120.0, zero_grads: bool = True):
        """One iteration; returns (loss tensor on device, raw events, t0)."""
        if zero_grads:
            for row in self.grid:
                for st in row:
                    st.zero_grads()
        events, t0s = self.group.run_iteration(watchdog_secs)
        self.last_events = (events, min(t0s))
        self.check_tp()
        last = self.stages[-1]
        return last.loss.sum() / (last.cfg.seq * self.M)

    def launch(self, zero_grads: bool = True):
        """Asynchronous step (for timing loops): enqueue, do not wait."""
        if zero_grads:
            for row in self.grid:
                for st in row:
                    st.zero_grads()
        self.group.launch()

    def wait(self, watchdog_secs: float = 120.0):
        events, t0s = self.group.wait(watchdog_secs)
        self.last_events = (events, min(t0s))
        self.check_tp()
        return events

    def nominal_us(self):
        """Per-stage mean F/B/W durations (µs) of the last iteration."""
        tr, _ = self.trace()
        return measured_nominal(tr, self.N)

    def set_nominal_latency(self, nominal_us):
        """Per-stage measured F/B/W means (µs, e.g. from nominal_us()) become the
        workload's latency table: the J-preset jitter pads then scale with the
        real task times instead of the construction-time placeholders."""
        from .workload import TaskId
        lat = {}
        for t in self.workload.latency:
            v = nominal_us[t.stage].get(t.direction, 0.0)
            lat[TaskId(t.stage, t.microbatch, t.chunk, t.direction)] = max(1, int(round(v)))
        self.group.set_latency(lat)
        self.workload = self.group.w

    def set_lognormal_jitter(self, sigma: float, seed: int = 0, nominal_us=None):
        """Enable injected lognormal compute jitter; nominal task times default
        to the last iteration's measured means (call after a clean step)."""
        if nominal_us is None:
            tr, _ = self.trace()
            nominal_us = measured_nominal(tr, self.N)
        self.nominal_table = nominal_us
        floors = lognormal_floor_tables(self.N, self.M, nominal_us, sigma, seed, n_chunks=self.C)
        self.group.set_floor_us(floors)

    def kernel_launches_per_step(self):
        """Our kernels launched per iteration: every task body (captured counts),
        one dispatcher step kernel per task plus the exiting step, and the
        lane's init / final kernels."""
        n = 0
        for row in self.grid:
            for st in row:
                n += sum(st.kernel_counts.values()) + len(st.kernel_counts)
        return n + 3 * self.N * self.R

    def trace(self):
        """(Trace, Metrics) of the last iteration: wall clock, or the virtual
        clock in replay mode (the lanes' own decisions at engine times)."""
        ev, t0 = self.last_events
        self.group.w = self.workload
        return self.group.make_trace(ev, [t0])

    def decisions(self):
        """Every arbitration the lanes evaluated in the last iteration
        (constructed with declog_cap > 0), for the per-decision oracle check."""
        return self.group.decisions()

    def check_tp(self):
        """A timed-out TP all-reduce only sets a sticky error word on the
        device (csrc/tp.cu): surface it as an exception after every step."""
        for s, comms in self.comms.items():
            for c in comms:
                if c.error():
                    raise RuntimeError(f"TP all-reduce of stage {s} rank {c.rank} timed out "
                                       "waiting for a peer: this iteration's results are invalid")

    def close(self):
        self.group.close()
        for comms in self.comms.values():
            for c in comms:
                c.close()
        self.comms = {}
        for row in self.grid or []:
            for st in row:
                st.release()
        self.grid = self.stages = None
        raw = getattr(self, "_green_raw", None)
        if raw is not None:     # the SM partitions of the single-GPU emulation
            from . import _lib
            torch.cuda.synchronize()
            self.green_streams = {}
            _lib.check(_lib.lib().rrfp_green_destroy(raw, len(raw) // 2))
            self._green_raw = None
