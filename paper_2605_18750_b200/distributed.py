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
    """Zero-copy torch view of raw device memory (bf16 via int16 typestr)."""
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaArray(ptr, shape, "<i2"), device=device)
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


def open_handle(handle: bytes) -> int:
    p = C.c_void_p()
    _lib.check(_lib.lib().rrfp_ipc_open(handle, C.byref(p)))
    return p.value


class DistPipeline:
    """This rank's stage of a PP=world pipeline (one stage per GPU)."""

    def __init__(self, cfg, n_mb: int, *, hint="bf", buffer_limit=32, mode="free", jitter=None,
                 seed=0, model_seed=1234, data_seed=0, schedule=None, group=None, comm_delay=None):
        import torch.distributed as dist
        from .arbitration import HintOrder
        from .model import StageCompute
        from .pipeline import nominal_workload
        from .runtime import LaneGroup
        if isinstance(hint, str):
            hint = HintOrder.parse(hint)
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.cuda.current_device()
        n, s = self.world, self.rank
        decompose = hint.kind == "bfw"
        S, D = cfg.seq, cfg.d_model
        slot_bytes = n_mb * S * D * 2
        self.bufs = {"fwd": IpcBuffer(slot_bytes, self.device) if s > 0 else None,
                     "bwd": IpcBuffer(slot_bytes, self.device) if s < n - 1 else None}
        fwd_in = wrap_bf16(self.bufs["fwd"].ptr.value, (n_mb, S, D), self.device) if s > 0 else None
        bwd_in = wrap_bf16(self.bufs["bwd"].ptr.value, (n_mb, S, D), self.device) if s < n - 1 else None
        self.stage = StageCompute(cfg, s, n, n_mb, torch.device("cuda", self.device),
                                  decompose=decompose, seed=model_seed, data_seed=data_seed,
                                  fwd_in=fwd_in, bwd_in=bwd_in)
        w = nominal_workload(cfg, n, n_mb, decompose)
        if comm_delay is not None:
            from .workload import Workload
            w = Workload(num_stages=n, num_microbatches=n_mb, num_chunks=1, tp_group_size=1,
                         latency=w.latency, comm_delay=comm_delay, decompose_backward=decompose)
        self.workload = w
        self.n_mb = n_mb
        self.group = LaneGroup(w, hint, buffer_limit, 1.0, seed=seed, jitter=jitter, mode=mode,
                               placement=[[self.device] for _ in range(n)], local=[(s, 0)],
                               bodies=None, compute_kind=1, schedule=schedule, defer_bodies=True)
        mine = {"stage": s, "fwd": self.bufs["fwd"].handle() if self.bufs["fwd"] else None,
                "bwd": self.bufs["bwd"].handle() if self.bufs["bwd"] else None,
                "lane": self.group.ipc_handles()[(s, 0)]}
        allh = [None] * n
        dist.all_gather_object(allh, mine, group=group)
        peers = plan_peers(s, n)
        fwd_out = bwd_out = None
        if peers["writes_fwd_mailbox"]:
            base = open_handle(allh[s + 1]["fwd"])
            fwd_out = wrap_bf16(base, (n_mb, S, D), self.device)
        if peers["writes_bwd_mailbox"]:
            base = open_handle(allh[s - 1]["bwd"])
            bwd_out = wrap_bf16(base, (n_mb, S, D), self.device)
        self.stage.connect_outputs(fwd_out=[fwd_out[mb] for mb in range(n_mb)] if fwd_out is not None else None,
                                   bwd_out=[bwd_out[mb] for mb in range(n_mb)] if bwd_out is not None else None)
        raw = self.stage.capture_bodies()
        self.group.set_bodies({(s, 0): raw})
        self.group.connect_ipc({(h["stage"], 0): h["lane"] for h in allh})
        torch.cuda.synchronize()
        dist.barrier(group=group)
        # every rank instantiates + uploads its lane graph before ANY rank launches
        self.group.prepare()
        dist.barrier(group=group)

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
            allv = [None] * self.world
            dist.all_gather_object(allv, mine, group=group)
            nominal_us = allv
        self.nominal_us = nominal_us
        floors = lognormal_floor_tables(self.world, self.n_mb, nominal_us, sigma, seed, stages=[self.rank])
        self.group.set_floor_us(floors)

    def kernel_launches_per_step(self):
        return sum(self.stage.kernel_counts.values()) + 2 * len(self.stage.kernel_counts) + 2

    def step(self, watchdog_secs=120.0):
        self.stage.zero_grads()
        events, t0s = self.group.run_iteration(watchdog_secs)
        self.last_events = (events, min(t0s))
        if self.stage.last:
            return self.stage.loss.sum() / (self.stage.cfg.seq * self.stage.M)
        return None

    def launch(self):
        self.stage.zero_grads()
        self.group.launch()

    def wait(self, watchdog_secs=120.0):
        events, t0s = self.group.wait(watchdog_secs)
        self.last_events = (events, min(t0s))
        return events

    def close(self):
        self.group.close()
