"""One process per GPU: each torchrun rank is one pipeline stage.

Wiring (no data-path collective -- the pipeline only has neighbour P2P):
  * every rank allocates its mailboxes (F-input and B-input slots, one per
    microbatch) and its lane inbox with cudaMalloc so they can be exported
    as CUDA IPC handles;
  * handles are exchanged ONCE with ``all_gather_object`` over the process
    group (plumbing only);
  * rank s opens rank s+1's F mailbox (its forward tasks write their output
    there), rank s-1's B mailbox, and every lane's inbox (flag stores +
    iteration barrier) -- after that all traffic is device-initiated NVLink
    stores + st.release.sys flags, no host round trip.

``plan_peers`` is the pure topology function (unit-tested on CPU with gloo).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib


def stage_coords(global_rank: int, world: int, tp_size: int = 1):
    """torchrun rank -> (pipeline stage, TP rank, n_stages): the TP ranks of a
    stage are adjacent process ranks (adjacent GPUs of the box)."""
    if tp_size < 1 or world % tp_size:
        raise ValueError(f"world size {world} is not a multiple of the TP size {tp_size}")
    return global_rank // tp_size, global_rank % tp_size, world // tp_size


def plan_peers(stage: int, n_stages: int, n_ranks: int = 1):
    """Who a lane sends to: F output -> next stage (chunk wrap to stage 0),
    B output -> previous stage (wrap to N-1); all R ranks of the receiver."""
    f_dst = stage + 1 if stage + 1 < n_stages else 0
    b_dst = stage - 1 if stage > 0 else n_stages - 1
    return {"fwd": [(f_dst, r) for r in range(n_ranks)],
            "bwd": [(b_dst, r) for r in range(n_ranks)],
            "writes_fwd_mailbox": stage + 1 < n_stages,
            "writes_bwd_mailbox": stage > 0}


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def wrap_bf16(ptr: int, shape, device) -> torch.Tensor:
    """Zero-copy torch view of raw device memory (bf16 via int16 typestr).

    No ``device=`` conversion: torch places a __cuda_array_interface__ tensor on
    the device that OWNS the pointer, and converting a peer GPU's mailbox to the
    local device would silently copy it (writes would land in the copy).  The
    kernels only use the address; the assert guards the zero-copy contract."""
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaArray(ptr, shape, "<i2"))
    if t.data_ptr() != ptr:
        raise RuntimeError("wrap_bf16: torch copied the buffer instead of viewing it")
    return t.view(torch.bfloat16)


class IpcBuffer:
    """A cudaMalloc'd buffer exportable through CUDA IPC."""

    def __init__(self, nbytes: int, device: int):
        L = _lib.lib()
        self.ptr = C.c_void_p()
        torch.cuda.set_device(device)
        _lib.check(L.rrfp_ipc_alloc(C.c_size_t(nbytes), C.byref(self.ptr)))
        self.nbytes, self.device = nbytes, device

    def handle(self) -> bytes:
        buf = (C.c_char * 64)()
        _lib.check(_lib.lib().rrfp_ipc_handle(self.ptr, buf))
        return bytes(buf)

    def free(self):
        if self.ptr:
            _lib.lib().rrfp_ipc_free(self.ptr)
            self.ptr = None


def open_handle(handle: bytes, track: list | None = None) -> int:
    """Map a peer's IPC buffer; `track` collects the pointer so the owner can
    unmap it (close_handles) when it is torn down."""
    p = C.c_void_p()
    _lib.check(_lib.lib().rrfp_ipc_open(handle, C.byref(p)))
    if track is not None:
        track.append(p.value)
    return p.value


def close_handles(ptrs: list):
    for ptr in ptrs:
        _lib.check(_lib.lib().rrfp_ipc_close(C.c_void_p(ptr)))
    ptrs.clear()


class DistPipeline:
    """This rank's lane of a PP x TP pipeline: one (stage, TP rank) per GPU.

    world = n_stages * tp_size; stage_coords() maps the process rank.  Every
    sender rank writes its output into the mailbox of EVERY TP rank of the
    neighbour stage (identical bytes), then raises its flags (runtime lane_send);
    TP partial sums are all-reduced over peer memory (tp.py / csrc/tp.cu)."""

    def __init__(self, cfg, n_mb: int, *, hint="bf", buffer_limit=32, mode="free", jitter=None,
                 seed=0, model_seed=1234, data_seed=0, schedule=None, group=None, comm_delay=None,
                 tp_size: int = 1, tp=None, n_chunks: int = 1, mm=None, head_cost: float = 0.0, w_split: str = "fc",
                 split: str = "layer"):
        import torch.distributed as dist
        from .arbitration import HintOrder, TpGroup
        from .model import StageCompute
        from .pipeline import nominal_workload
        from .runtime import LaneGroup
        if isinstance(hint, str):
            hint = HintOrder.parse(hint)
        self.grank, self.gworld = dist.get_rank(group), dist.get_world_size(group)
        s, r, n = stage_coords(self.grank, self.gworld, tp_size)
        R, C = tp_size, n_chunks
        V = n * C
        if mm is not None and (R > 1 or C > 1):
            raise ValueError("the multimodal pipeline (config 4) runs with TP=1, C=1")
        stage_cfg = (lambda v: mm.vit if v < mm.vit_stages else mm.llm) if mm else (lambda v: cfg)
        self.rank, self.world, self.tp_rank, self.R, self.C = s, n, r, R, C
        self.device = torch.cuda.current_device()
        decompose = hint.kind == "bfw"
        # this lane hosts virtual stages v = c*N + s (chunk c), each with its own mailboxes:
        # F input [M, S, D] of the stage's own width; B input [M, S, D_out] (the ViT
        # projector stage receives the gradient of its d_llm-wide output)
        self.vids = [c * n + s for c in range(C)]
        self.bufs, shapes = {}, {}
        for v in self.vids:
            vc = stage_cfg(v)
            d_out = mm.llm.d_model if (mm and v == mm.vit_stages - 1) else vc.d_model
            shapes[v] = ((n_mb, vc.seq, vc.d_model), (n_mb, vc.seq, d_out))
            self.bufs[(v, "fwd")] = IpcBuffer(2 * n_mb * vc.seq * vc.d_model, self.device) if v > 0 else None
            self.bufs[(v, "bwd")] = IpcBuffer(2 * n_mb * vc.seq * d_out, self.device) if v < V - 1 else None
        self.comm = None
        if R > 1:
            from .tp import TpComm
            self.comm = TpComm(r, R, (cfg.seq, cfg.d_model), torch.device("cuda", self.device))
        self.clock_slot = IpcBuffer(16, self.device)      # cross-GPU timer calibration
        self._opened = []                                 # peer buffers this rank mapped
        self.clock_offset_ns = 0                          # this rank's clock - rank 0's clock
        self.vstages = []
        for v in self.vids:
            fb, bb = self.bufs[(v, "fwd")], self.bufs[(v, "bwd")]
            self.vstages.append(StageCompute(
                stage_cfg(v), v, V, n_mb, torch.device("cuda", self.device), decompose=decompose,
                seed=model_seed, data_seed=data_seed,
                fwd_in=wrap_bf16(fb.ptr.value, shapes[v][0], self.device) if fb else None,
                bwd_in=wrap_bf16(bb.ptr.value, shapes[v][1], self.device) if bb else None,
                tp_rank=r, tp_size=R, tp=self.comm, mm=mm, head_cost=head_cost if C == 1 else 0.0,
                w_split=w_split, split=split))
        # the lane's first / last virtual stages (loss lives on virtual stage V-1)
        self.stage = self.vstages[-1] if self.vstages[-1].last else self.vstages[0]
        w = nominal_workload(cfg, n, n_mb, decompose, tp_size=R, n_chunks=C)
        if comm_delay is not None:
            from .workload import Workload
            w = Workload(num_stages=n, num_microbatches=n_mb, num_chunks=C, tp_group_size=R,
                         latency=w.latency, comm_delay=comm_delay, decompose_backward=decompose)
        self.workload = w
        self.n_mb = n_mb
        self.group = LaneGroup(w, hint, buffer_limit, 1.0, seed=seed, jitter=jitter, mode=mode,
                               tp=tp or (TpGroup(group_size=R) if R > 1 else None),
                               placement=[[self.device] * R for _ in range(n)], local=[(s, r)],
                               bodies=None, compute_kind=1, schedule=schedule, defer_bodies=True)
        hd = lambda b: b.handle() if b else None
        mine = {"stage": s, "tp_rank": r,
                "mbox": {v: (hd(self.bufs[(v, "fwd")]), hd(self.bufs[(v, "bwd")]), shapes[v]) for v in self.vids},
                "lane": self.group.ipc_handles()[(s, r)],
                "tp": self.comm.ipc_handles() if self.comm else None,
                "clock": self.clock_slot.handle(),
                "gpu_uuid": str(torch.cuda.get_device_properties(self.device).uuid)}
        allh = [None] * self.gworld
        dist.all_gather_object(allh, mine, group=group)
        by = {(h["stage"], h["tp_rank"]): h for h in allh}
        self._clock_peers = [h["clock"] for h in allh]     # by global rank
        self._gpu_uuid = [h["gpu_uuid"] for h in allh]
        self._group = group
        if self.comm:
            self.comm.connect_ipc([by[(s, q)]["tp"] for q in range(R)])

        def mailboxes(v, which):   # virtual stage v's F (0) / B (1) mailbox on every TP rank
            dst = [wrap_bf16(open_handle(by[(v % n, q)]["mbox"][v][which], self._opened),
                             by[(v % n, q)]["mbox"][v][2][which], self.device) for q in range(R)]
            return [[d[mb] for d in dst] for mb in range(n_mb)]

        for st, v in zip(self.vstages, self.vids):
            st.connect_outputs(fwd_out=mailboxes(v + 1, 0) if v + 1 < V else None,
                               bwd_out=mailboxes(v - 1, 1) if v > 0 else None)
        # eager warm-up with rank-local all-reduces (module loading never races a spinning peer)
        if self.comm:
            self.comm.local_only = True
        for st in self.vstages:
            st.warmup().synchronize()
        if self.comm:
            self.comm.local_only = False
        arr = [None] * (3 * n_mb * C)
        for c, st in enumerate(self.vstages):
            raw = st.capture()
            for ki in range(3):
                for mb in range(n_mb):
                    arr[ki * n_mb * C + c * n_mb + mb] = raw[ki * n_mb + mb]
        self.group.set_bodies({(s, r): arr})
        self.group.connect_ipc({(h["stage"], h["tp_rank"]): h["lane"] for h in allh})
        torch.cuda.synchronize()
        dist.barrier(group=group)
        # every rank instantiates + uploads its lane graph before ANY rank launches
        self.group.prepare()
        dist.barrier(group=group)

    def calibrate_clocks(self, rounds: int = 16, force: bool = False):
        """Offsets of every rank's %globaltimer against rank 0's (ping-pong over
        peer memory, one pair at a time); afterwards ``clock_offset_ns`` maps this
        rank's device timestamps onto rank 0's clock (subtract it).  Collective.
        Ranks on the same GPU share one timer (offset 0) unless ``force`` (tests).
        Returns (offset_ns, best_rtt_ns) of this rank ((0, 0) on rank 0)."""
        import ctypes as C
        import torch.distributed as dist
        L = _lib.lib()
        me = self.grank
        measured = {}
        calls = self._clock_calls = getattr(self, "_clock_calls", 0) + 1   # same count on every rank
        for peer in range(1, self.gworld):
            dist.barrier(group=self._group)
            if me not in (0, peer):
                continue
            if not force and self._gpu_uuid[peer] == self._gpu_uuid[0]:   # same GPU: one timer
                if me == 0:
                    measured[peer] = (0, 0)
                continue
            other = peer if me == 0 else 0
            opened = self.__dict__.setdefault("_clock_opened", {})
            if other not in opened:
                opened[other] = open_handle(self._clock_peers[other], self._opened)
            ptr = opened[other]
            o, t = C.c_longlong(), C.c_longlong()
            base = (calls * self.gworld + peer) * (rounds + 1)   # round ids grow on every slot
            _lib.check(L.rrfp_clock_pingpong(self.clock_slot.ptr, C.c_void_p(ptr), 0 if me == 0 else 1, rounds,
                                             C.c_longlong(base), C.byref(o), C.byref(t)))
            if me == 0:
                measured[peer] = (o.value, t.value)
        table = [measured if me == 0 else None]       # rank 0 hands every rank its offset
        dist.broadcast_object_list(table, src=0, group=self._group)
        off, rtt = table[0].get(me, (0, 0))
        self.clock_offset_ns = off
        return off, rtt

    def aligned_events(self):
        """The last iteration's device events as tuples (t0, t1, kind, stage, rank,
        task) on rank 0's clock (see calibrate_clocks), and the aligned t0."""
        ev, t0 = self.last_events
        d = self.clock_offset_ns
        return [(e.t0 - d, e.t1 - d, e.kind, e.stage, e.rank, e.task) for e in ev], t0 - d

    def nominal_us(self, group=None):
        """Per-stage mean F/B/W durations (µs) of the last iteration, gathered
        from TP rank 0 of every stage (collective: call on every rank)."""
        import torch.distributed as dist
        ev, _ = self.last_events
        mine = {}
        for d, code in (("F", 1), ("B", 0), ("W", 2)):
            xs = [e.t1 - e.t0 for e in ev if e.kind == 0 and (e.task & 3) == code]
            mine[d] = (sum(xs) / len(xs) / 1000.0) if xs else 0.0
        allv = [None] * self.gworld
        dist.all_gather_object(allv, mine, group=group)
        return allv[::self.R]

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

    def set_lognormal_jitter(self, sigma: float, seed: int = 0, nominal_us=None, group=None):
        """Lognormal compute jitter floors for THIS rank's stage; nominal task
        times are gathered from every rank's last iteration."""
        import torch.distributed as dist
        from .pipeline import lognormal_floor_tables
        if nominal_us is None:
            ev, _ = self.last_events
            mine = {}
            for d, code in (("F", 1), ("B", 0), ("W", 2)):
                xs = [e.t1 - e.t0 for e in ev if e.kind == 0 and (e.task & 3) == code]
                mine[d] = (sum(xs) / len(xs) / 1000.0) if xs else 0.0
            allv = [None] * self.gworld
            dist.all_gather_object(allv, mine, group=group)
            nominal_us = allv[::self.R]      # TP rank 0 of every stage
        self.nominal_table = nominal_us
        floors = lognormal_floor_tables(self.world, self.n_mb, nominal_us, sigma, seed, stages=[self.rank],
                                        n_chunks=self.C)
        self.group.set_floor_us(floors)

    def kernel_launches_per_step(self):
        # bodies + one dispatcher step per task, the exiting step, init and final
        return sum(sum(st.kernel_counts.values()) + len(st.kernel_counts) for st in self.vstages) + 3

    def step(self, watchdog_secs=120.0):
        for st in self.vstages:
            st.zero_grads()
        events, t0s = self.group.run_iteration(watchdog_secs)
        self.last_events = (events, min(t0s))
        self.check_tp()
        if self.stage.last:
            return self.stage.loss.sum() / (self.stage.cfg.seq * self.stage.M)
        return None

    def launch(self):
        for st in self.vstages:
            st.zero_grads()
        self.group.launch()

    def wait(self, watchdog_secs=120.0):
        events, t0s = self.group.wait(watchdog_secs)
        self.last_events = (events, min(t0s))
        self.check_tp()
        return events

    def check_tp(self):
        """Raise if this rank's TP all-reduce timed out on a peer (csrc/tp.cu
        only sets a sticky error word on the device)."""
        if self.comm is not None and self.comm.error():
            raise RuntimeError(f"TP all-reduce of stage {self.rank} rank {self.tp_rank} timed out "
                               "waiting for a peer: this iteration's results are invalid")

    def close(self):
        self.group.close()
        if self.comm:
            self.comm.close()
            self.comm = None
        close_handles(self._opened)
        self.__dict__.pop("_clock_opened", None)
        for st in self.vstages or []:
            st.release()
        self.vstages = []
        self.stage = None
        for b in self.bufs.values():
            if b is not None:
                b.free()
        self.bufs = {}
        if self.clock_slot is not None:
            self.clock_slot.free()
            self.clock_slot = None
