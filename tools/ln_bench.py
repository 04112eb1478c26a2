"""LayerNorm-backward variants on the GPT-1.3B shape [2048 x 2048] (dev tool):
the separate kernels the B body ran in round 1 (dx + parameter gradients +
two bias column sums) vs the one-pass fused kernel; CUDA events, 200 reps,
interleaved, medians.  Operands L2-resident as inside the B body."""
import ctypes as C
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import _lib

L = _lib.lib()
R, D = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 2048)))
bf = torch.bfloat16
x, dy, dres = (torch.randn(R, D, device="cuda").to(bf) for _ in range(3))
g = torch.ones(D, device="cuda").to(bf)
mean, rstd = torch.zeros(R, device="cuda"), torch.ones(R, device="cuda")
dx = torch.empty_like(x)
dg, db, c1, c2 = (torch.zeros(D, device="cuda") for _ in range(4))
p = lambda t: C.c_void_p(0 if t is None else t.data_ptr())
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)


def separate():
    L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), p(g), p(dres), p(dx), None, None, R, D, st())
    L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), None, None, None, p(dg), p(db), R, D, st())
    L.rrfp_bias_grad(p(dres), C.c_longlong(D), p(c1), R, D, st())
    L.rrfp_bias_grad(p(dx), C.c_longlong(D), p(c2), R, D, st())


def dx_only():
    L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), p(g), p(dres), p(dx), None, None, R, D, st())


def fused():
    L.rrfp_layernorm_bwd_fused(p(dy), p(x), p(mean), p(rstd), p(g), p(dres), p(dx), p(dg), p(db), p(c1), p(c2),
                               R, D, st())


def fused_dx_only():
    L.rrfp_layernorm_bwd_fused(p(dy), p(x), p(mean), p(rstd), p(g), p(dres), p(dx), None, None, None, None,
                               R, D, st())


def t(fn, reps=200):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def side_separate():
    L.rrfp_layernorm_bwd(p(dy), p(x), p(mean), p(rstd), None, None, None, p(dg), p(db), R, D, st())
    L.rrfp_bias_grad(p(dres), C.c_longlong(D), p(c1), R, D, st())


def side_fused():
    L.rrfp_layernorm_bwd_fused(p(dy), p(x), p(mean), p(rstd), None, p(dres), None, p(dg), p(db), p(c1), None,
                               R, D, st())


V = [("separate (dx + params + 2 colsums)", separate), ("dx only (ln_bwd_dx)", dx_only),
     ("fused (all five outputs)", fused), ("fused, dx only", fused_dx_only),
     ("side: params + colsum(dres), 2 kernels", side_separate), ("side: fused params + colsum(dres)", side_fused)]
for _, fn in V:
    t(fn, 50)
res = {n: [] for n, _ in V}
for _ in range(10):
    for n, fn in V:
        res[n].append(t(fn))
byt = 4 * R * D * 2   # dy, x, dres read + dx written (bf16)
print(f"# LN backward [{R} x {D}] bf16, one B200, medians of 10 x 200 launches")
for n, _ in V:
    m = statistics.median(res[n])
    print(f"{n:38s} {m:7.2f} us   {byt / m / 1e3:7.0f} GB/s (dy + x + dres + dx bytes)")
