"""Run one layer's epilogue-heavy GEMMs once each (for ncu --set full)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import kernels as K
S, D, F = 2048, 2048, 8192
bf = torch.bfloat16
r = lambda *s: torch.randn(*s, device="cuda").to(bf)
x, w1, w2, wo = r(S, D), r(F, D), r(D, F), r(D, D)
b1, bd = r(F), r(D)
pre, act, y, dpre = (torch.empty(S, F, device="cuda", dtype=bf), torch.empty(S, F, device="cuda", dtype=bf),
                     torch.empty(S, D, device="cuda", dtype=bf), torch.empty(S, F, device="cuda", dtype=bf))
g1 = torch.zeros(F, D, device="cuda")
calls = [lambda: K.gemm(x, w1, pre, epi=K.EPI_BIAS_GELU, c2=act, bias=b1),          # fc1 fwd
         lambda: K.gemm(x, w2, dpre, epi=K.EPI_GELU_BWD, b_mn=True, r=pre),        # fc2 dgrad
         lambda: K.gemm(x, wo, y, epi=K.EPI_RESID, bias=bd, r=x),                   # proj fwd
         lambda: K.gemm(dpre, x, g1, epi=K.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True)]  # fc1 wgrad
for _ in range(3):
    for c in calls: c()
torch.cuda.synchronize()
for c in calls: c()
torch.cuda.synchronize()
print("done")
