"""CUDA-event timing of the HBM-bound stage ops at GPT-1.3B shapes (dev tool):
achieved GB/s against the algorithmic bytes."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import _lib

L = _lib.lib()
p = lambda t: C.c_void_p(0 if t is None else t.data_ptr())
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)


def t(fn, reps=20):
    """Per-launch device time of `reps` back-to-back launches captured in one CUDA
    graph (as in the task bodies: no host launch overhead between them)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(reps): fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


S, D, V = 2048, 2048, 50304
logits = torch.randn(S, V, device="cuda").bfloat16()
tgt = torch.randint(0, V, (S,), device="cuda", dtype=torch.int32)
loss, lse = torch.empty(S, device="cuda"), torch.empty(S, device="cuda")
us = t(lambda: L.rrfp_xent_fwd(p(logits), C.c_longlong(V), p(tgt), S, V, p(loss), p(lse), st()))
print(f"xent_fwd  [2048 x 50304]: {us:6.1f} us  {S * V * 2 / us / 1e3:6.0f} GB/s")
x = torch.randn(S, D, device="cuda").bfloat16()
dy = torch.randn(S, D, device="cuda").bfloat16()
g = torch.ones(D, device="cuda").bfloat16()
b = torch.zeros(D, device="cuda").bfloat16()
y = torch.empty_like(x)
mean, rstd = torch.empty(S, device="cuda"), torch.empty(S, device="cuda")
us = t(lambda: L.rrfp_layernorm_fwd(p(x), p(g), p(b), p(y), p(mean), p(rstd), S, D, C.c_float(1e-5), st()))
print(f"ln_fwd    [2048 x 2048]:  {us:6.1f} us  {2 * S * D * 2 / us / 1e3:6.0f} GB/s")
dx = torch.empty_like(x)
dg, db = torch.zeros(D, device="cuda"), torch.zeros(D, device="cuda")
us = t(lambda: L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), p(g), p(dy), p(dx), None, None, S, D, st()))
print(f"ln_bwd dx [2048 x 2048]:  {us:6.1f} us  {4 * S * D * 2 / us / 1e3:6.0f} GB/s")
us = t(lambda: L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), p(g), None, None, p(dg), p(db), S, D, st()))
print(f"ln_bwd dg [2048 x 2048]:  {us:6.1f} us  {2 * S * D * 2 / us / 1e3:6.0f} GB/s")
for cols in (2048, 6144, 8192):
    a = torch.randn(S, cols, device="cuda").bfloat16()
    o = torch.zeros(cols, device="cuda")
    us = t(lambda: L.rrfp_bias_grad(p(a), C.c_longlong(cols), p(o), S, cols, st()))
    print(f"colsum    [2048 x {cols}]:  {us:6.1f} us  {S * cols * 2 / us / 1e3:6.0f} GB/s")
