"""Attention core of the stage bodies: cuDNN SDPA (library, SURVEY.md K9
"library first") driven through the cuDNN frontend graph API.

Going through the graph API instead of ``aten._scaled_dot_product_cudnn_attention``
lets every tensor have the stride we store it with:

  * Q, K, V are read straight out of the packed QKV GEMM output [T, 3·D]
    (head-major columns, row stride 3·D);
  * O is written into the stage's own activation slot [T, D] and the softmax
    statistics into its own fp32 slot [H, S_max];
  * dQ, dK, dV are written straight into the packed gradient [T, 3·D] that the
    QKV dgrad / wgrad GEMMs consume -- the torch op allocates three separate
    tensors that had to be copied in (3 copy kernels on the B chain).

One graph pair per (T, heads, head_dim, causal, device), built once and
executed with per-call pointers (capturable in the stage's CUDA graphs); the
workspace is owned by the caller (stages that may run concurrently on one GPU
never share it).  No fallback: a missing cuDNN frontend raises.
"""

from __future__ import annotations

import math

import torch

_HANDLES = {}
_GRAPHS = {}


def _handle(device: torch.device):
    import cudnn
    key = device.index
    if key not in _HANDLES:
        with torch.cuda.device(device):
            _HANDLES[key] = cudnn.create_handle()
    return _HANDLES[key]


class SdpaGraphs:
    """Forward + backward cuDNN graphs for one attention shape."""

    def __init__(self, T: int, H: int, Dh: int, causal: bool, device, stats_row: int):
        import cudnn
        self.T, self.H, self.Dh, self.causal = T, H, Dh, causal
        self.device = torch.device(device)
        D = H * Dh
        self.D = D
        bf, f32 = cudnn.data_type.BFLOAT16, cudnn.data_type.FLOAT
        h = _handle(self.device)
        self.handle = h
        scale = 1.0 / math.sqrt(Dh)
        dim = [1, H, T, Dh]
        qkv_stride = [T * 3 * D, Dh, 3 * D, 1]
        o_stride = [T * D, Dh, D, 1]
        st_dim, st_stride = [1, H, T, 1], [H * stats_row, stats_row, 1, 1]
        plans = [cudnn.heur_mode.A, cudnn.heur_mode.FALLBACK]

        def build(g):
            g.validate()
            g.build_operation_graph()
            g.create_execution_plans(plans)
            g.check_support()
            g.build_plans()

        with torch.cuda.device(self.device):
            g = cudnn.pygraph(io_data_type=bf, intermediate_data_type=f32, compute_data_type=f32, handle=h)
            q = g.tensor(name="q", dim=dim, stride=qkv_stride, data_type=bf)
            k = g.tensor(name="k", dim=dim, stride=qkv_stride, data_type=bf)
            v = g.tensor(name="v", dim=dim, stride=qkv_stride, data_type=bf)
            o, stats = g.sdpa(name="sdpa", q=q, k=k, v=v, generate_stats=True, attn_scale=scale,
                              use_causal_mask=causal)
            o.set_output(True).set_dim(dim).set_stride(o_stride).set_data_type(bf)
            stats.set_output(True).set_dim(st_dim).set_stride(st_stride).set_data_type(f32)
            build(g)
            self.fwd_graph, self.f = g, (q, k, v, o, stats)

            b = cudnn.pygraph(io_data_type=bf, intermediate_data_type=f32, compute_data_type=f32, handle=h)
            bq = b.tensor(name="q", dim=dim, stride=qkv_stride, data_type=bf)
            bk = b.tensor(name="k", dim=dim, stride=qkv_stride, data_type=bf)
            bv = b.tensor(name="v", dim=dim, stride=qkv_stride, data_type=bf)
            bo = b.tensor(name="o", dim=dim, stride=o_stride, data_type=bf)
            bdo = b.tensor(name="do", dim=dim, stride=o_stride, data_type=bf)
            bst = b.tensor(name="stats", dim=st_dim, stride=st_stride, data_type=f32)
            dq, dk, dv = b.sdpa_backward(name="sdpa_bwd", q=bq, k=bk, v=bv, o=bo, dO=bdo, stats=bst,
                                         attn_scale=scale, use_causal_mask=causal)
            for t in (dq, dk, dv):
                t.set_output(True).set_dim(dim).set_stride(qkv_stride).set_data_type(bf)
            build(b)
            self.bwd_graph, self.b = b, (bq, bk, bv, bo, bdo, bst, dq, dk, dv)
        self.workspace_bytes = max(self.fwd_graph.get_workspace_size(), self.bwd_graph.get_workspace_size())

    def forward(self, qkv_ptr: int, o_ptr: int, stats_ptr: int, ws_ptr: int, stream: int):
        import cudnn
        q, k, v, o, st = self.f
        e = 2 * self.D
        cudnn.set_stream(handle=self.handle, stream=stream)
        self.fwd_graph.execute({q: qkv_ptr, k: qkv_ptr + e, v: qkv_ptr + 2 * e, o: o_ptr, st: stats_ptr},
                               ws_ptr, handle=self.handle)

    def backward(self, qkv_ptr: int, o_ptr: int, do_ptr: int, stats_ptr: int, dqkv_ptr: int, ws_ptr: int,
                 stream: int):
        import cudnn
        q, k, v, o, do, st, dq, dk, dv = self.b
        e = 2 * self.D
        cudnn.set_stream(handle=self.handle, stream=stream)
        self.bwd_graph.execute({q: qkv_ptr, k: qkv_ptr + e, v: qkv_ptr + 2 * e, o: o_ptr, do: do_ptr,
                                st: stats_ptr, dq: dqkv_ptr, dk: dqkv_ptr + e, dv: dqkv_ptr + 2 * e},
                               ws_ptr, handle=self.handle)


def sdpa_graphs(T: int, H: int, Dh: int, causal: bool, device, stats_row: int) -> SdpaGraphs:
    key = (T, H, Dh, bool(causal), torch.device(device).index, stats_row)
    if key not in _GRAPHS:
        _GRAPHS[key] = SdpaGraphs(T, H, Dh, causal, device, stats_row)
    return _GRAPHS[key]
