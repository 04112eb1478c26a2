"""ctypes front-end of the stage-compute kernels (csrc/*.cu) on torch tensors.

All entry points take torch CUDA tensors, pass raw device pointers through
the C ABI and launch on torch's current stream (so torch.cuda.graph capture
records them).  No fallback: a missing library raises.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib

EPI_BF16, EPI_BIAS_GELU, EPI_RESID, EPI_ACC_F32, EPI_GELU_BWD, EPI_F32, EPI_BF16_LSE = range(7)

# number of our own kernel launches issued through this module (graph bodies
# count them at capture time; bench.py reports launches per step)
LAUNCHES = [0]


def note(n: int = 1):
    LAUNCHES[0] += n


def _p(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ld(t, mn_major=False):
    return t.stride(0)


def gemm(a, b, c, *, epi=EPI_BF16, a_mn=False, b_mn=False, c2=None, bias=None, r=None,
         accumulate=False, m=None, n=None, k=None, ldc2=None):
    """c = op(a) . op(b)^T with fused epilogue (see csrc/gemm_sm100.cu).

    a: [M, K] (or [K, M] if a_mn); b: [N, K] (or [K, N] if b_mn); row-major, unit inner stride.
    """
    M = m if m is not None else (a.shape[1] if a_mn else a.shape[0])
    K = k if k is not None else (a.shape[0] if a_mn else a.shape[1])
    N = n if n is not None else (b.shape[1] if b_mn else b.shape[0])
    L = _lib.lib()
    note()
    _lib.check(L.rrfp_gemm_bf16(
        epi, int(a_mn), int(b_mn), M, N, K, _p(a), C.c_longlong(a.stride(0)), _p(b),
        C.c_longlong(b.stride(0)), _p(c), C.c_longlong(c.stride(0)), _p(c2),
        C.c_longlong(ldc2 if ldc2 is not None else (c2.stride(0) if c2 is not None else 0)), _p(bias), _p(r),
        C.c_longlong(r.stride(0) if r is not None else 0), int(accumulate), _stream()))
    return c


def attn_fwd(qkv, o, lse, *, heads, causal=True, scale=None, T=None):
    """Flash attention forward (csrc/fmha_sm100.cu): qkv [T, >=3D] packed, o [T, >=D],
    lse fp32 [H, >=T] (log2 units).  d_head = 128."""
    T = qkv.shape[0] if T is None else T
    dh = 128
    scale = dh ** -0.5 if scale is None else scale
    L = _lib.lib()
    note()
    _lib.check(L.rrfp_attn_fwd(_p(qkv), C.c_longlong(qkv.stride(0)), _p(o), C.c_longlong(o.stride(0)),
                               _p(lse), C.c_longlong(lse.stride(0)), T, heads, dh, int(causal),
                               C.c_float(scale), _stream()))
    return o


def attn_bwd_workspace(T, heads, device="cuda"):
    n = _lib.lib().rrfp_attn_bwd_workspace_bytes(T, heads)
    return torch.empty(n, device=device, dtype=torch.uint8)


def attn_bwd(qkv, o, do, lse, dqkv, ws, *, heads, causal=True, scale=None, T=None):
    """Flash attention backward (csrc/fmha_sm100.cu): dQ, dK, dV into the packed dqkv
    [T, >=3D]; lse = the forward's statistics [H, >=T]; ws from attn_bwd_workspace."""
    T = qkv.shape[0] if T is None else T
    dh = 128
    scale = dh ** -0.5 if scale is None else scale
    L = _lib.lib()
    note(4)
    _lib.check(L.rrfp_attn_bwd(_p(qkv), C.c_longlong(qkv.stride(0)), _p(o), C.c_longlong(o.stride(0)), _p(do),
                               C.c_longlong(do.stride(0)), _p(lse), C.c_longlong(lse.stride(0)), _p(dqkv),
                               C.c_longlong(dqkv.stride(0)), _p(ws), T, heads, dh, int(causal), C.c_float(scale),
                               _stream()))
    return dqkv


def lm_head_xent_fwd(hf, w_lm, logits, targets, loss, lse, part, *, rows=None):
    """LM head + cross-entropy forward: logits = hf . w_lm^T (bf16,
    tcgen05 GEMM) whose epilogue also emits each row's online-softmax
    statistics per 128-column slot into `part` (fp32 [rows, slots, 2]); a
    one-warp-per-row merge then gives lse and loss = lse - logit[target].  The
    logits are written once and not re-read in the forward."""
    rows = hf.shape[0] if rows is None else rows
    V = w_lm.shape[0]
    slots = part.shape[1]
    gemm(hf, w_lm, logits, epi=EPI_BF16_LSE, c2=part, ldc2=part.stride(0) // 2, m=rows, n=V, k=hf.shape[1])
    L = _lib.lib()
    note()
    _lib.check(L.rrfp_xent_combine(_p(part), C.c_longlong(part.stride(0) // 2), slots, _p(logits),
                                   C.c_longlong(logits.stride(0)), _p(targets), rows, _p(loss), _p(lse),
                                   _stream()))


def lm_head_slots(vocab):
    """float2 slots per row of lm_head_xent_fwd's statistics buffer."""
    return 2 * ((vocab + 255) // 256)
