import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_18750_b200 import kernels as K
S, D, F = 2048, 2048, 8192
bf = torch.bfloat16
dy = torch.randn(S, D, device="cuda").to(bf); w2 = torch.randn(D, F, device="cuda").to(bf)
pre = torch.randn(S, F, device="cuda").to(bf); out = torch.empty(S, F, device="cuda", dtype=bf)
cs = torch.zeros(F, device="cuda")
from paper_2605_18750_b200 import _lib
L = _lib.lib()
import ctypes as C
def a(): K.gemm(dy, w2, out, epi=K.EPI_GELU_BWD, b_mn=True, r=pre)
def b(): K.gemm(dy, w2, out, epi=K.EPI_GELU_BWD, b_mn=True, r=pre, c2=cs)
def c():
    K.gemm(dy, w2, out, epi=K.EPI_GELU_BWD, b_mn=True, r=pre)
    L.rrfp_bias_grad(C.c_void_p(out.data_ptr()), C.c_longlong(F), C.c_void_p(cs.data_ptr()), S, F, C.c_void_p(torch.cuda.current_stream().cuda_stream))
def t(fn, n=30):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n * 1e3
for f in (a, b, c): t(f, 50)
res = {k: [] for k in "abc"}
for _ in range(10):
    for k, f in zip("abc", (a, b, c)): res[k].append(t(f))
print("fc2 dgrad gelu' alone %.1f us | + colsum in epilogue %.1f us | + separate colsum kernel %.1f us" % tuple(statistics.median(res[k]) for k in "abc"))
