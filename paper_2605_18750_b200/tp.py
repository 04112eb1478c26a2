"""Tensor-parallel group of one pipeline stage (BASELINE config 3: TP=2 x PP=4).

``TpComm`` wraps the C-ABI TP group of csrc/tp.cu: a per-rank partial buffer
(the row-parallel GEMM writes its [S, D] partial sum there), a flag board the
peers write into, and ``allreduce`` -- one kernel that sums every rank's
partial in rank order over peer memory (NVLink when the ranks are on different
GPUs), fuses the row-parallel bias and the residual add, and stores the result
into up to four destinations.  The TP *agreement* (which task runs next) is
done by the lane dispatchers (tp_coordinate, arbitration.py:323-334); the
all-reduces of a task therefore happen in the same order on every rank.

Wiring:
  * one process, several ranks: ``connect_local([comm_0, comm_1, ...])``;
  * one process per GPU: ``ipc_handles()`` -> all_gather -> ``connect_ipc``.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from . import kernels as K


class TpComm:
    def __init__(self, rank: int, size: int, part_shape, device):
        self.rank, self.size = rank, size
        self.device = torch.device(device)
        self.part_shape = tuple(part_shape)
        nbytes = 2
        for s in self.part_shape:
            nbytes *= s
        L = _lib.lib()
        self.h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.rrfp_tp_create(rank, size, C.c_size_t(nbytes), C.byref(self.h)))
        part, board = C.c_void_p(), C.c_void_p()
        _lib.check(L.rrfp_tp_buffers(self.h, C.byref(part), C.byref(board)))
        self.part_ptr, self.board_ptr = part.value, board.value
        from .distributed import wrap_bf16
        self.partial = wrap_bf16(self.part_ptr, self.part_shape, self.device)
        # warm-up mode: all-reduces run rank-locally (no rendezvous), see rrfp_tp_allreduce
        self.local_only = False

    # ------------------------------------------------------------- wiring
    def connect(self, parts, boards):
        L = _lib.lib()
        pa = (C.c_void_p * self.size)(*parts)
        bo = (C.c_void_p * self.size)(*boards)
        _lib.check(L.rrfp_tp_connect(self.h, pa, bo))

    @staticmethod
    def connect_local(comms):
        parts = [c.part_ptr for c in comms]
        boards = [c.board_ptr for c in comms]
        for c in comms:
            c.connect(parts, boards)

    def ipc_handles(self):
        L = _lib.lib()
        a, b = (C.c_char * 64)(), (C.c_char * 64)()
        _lib.check(L.rrfp_ipc_handle(C.c_void_p(self.part_ptr), a))
        _lib.check(L.rrfp_ipc_handle(C.c_void_p(self.board_ptr), b))
        return bytes(a), bytes(b)

    def connect_ipc(self, handles):
        """handles[q] = (partial handle, board handle) of TP rank q (own included)."""
        from .distributed import open_handle
        parts, boards = [], []
        self._opened = getattr(self, "_opened", [])
        for q, (ph, bh) in enumerate(handles):
            if q == self.rank:
                parts.append(self.part_ptr)
                boards.append(self.board_ptr)
            else:
                parts.append(open_handle(ph, self._opened))
                boards.append(open_handle(bh, self._opened))
        self.connect(parts, boards)

    # ---------------------------------------------------------- collective
    def allreduce(self, outs, bias=None, resid=None):
        """outs[k] <- sum_q partial_q + bias + resid, for every destination in
        ``outs`` (tensors or RawBuffers of the partial's shape)."""
        rows, cols = self.part_shape
        ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        K.note()
        _lib.check(_lib.lib().rrfp_tp_allreduce(
            self.h, rows, cols, K._p(bias), K._p(resid),
            C.c_longlong(resid.stride(0) if resid is not None else 0), ptrs, len(outs),
            int(self.local_only), K._stream()))

    def error(self) -> int:
        e = C.c_int()
        _lib.check(_lib.lib().rrfp_tp_error(self.h, C.byref(e)))
        return e.value

    def close(self):
        from .distributed import close_handles
        close_handles(getattr(self, "_opened", []))
        if self.h:
            _lib.lib().rrfp_tp_destroy(self.h)
            self.h = None
