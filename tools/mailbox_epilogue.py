"""The stage's last F GEMM writes the next stage's mailbox slot.  On separate
GPUs that slot is peer memory, which takes the staged coalesced-store epilogue
(rrfp_gemm_set_epilogue(2)) instead of the TMA store; this times both on the
FC2 (+bias +residual) shape and reports the output write rate (dev tool; one
GPU, so the "peer" is local HBM here)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import _lib, kernels as K

L = _lib.lib()
S, D, F = 2048, 2048, 8192
act = torch.randn(S, F, device="cuda").bfloat16()
w2 = (torch.randn(D, F, device="cuda") * 0.02).bfloat16()
b2 = torch.zeros(D, device="cuda").bfloat16()
x2 = torch.randn(S, D, device="cuda").bfloat16()
out = torch.empty(S, D, device="cuda", dtype=torch.bfloat16)


def t(reps=30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        K.gemm(act, w2, out, epi=K.EPI_RESID, bias=b2, r=x2, m=S, n=D, k=F)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


res = {1: [], 2: []}
for _ in range(3):
    for v in (1, 2):
        L.rrfp_gemm_set_epilogue(v); t(5)
for _ in range(8):
    for v in (1, 2):
        L.rrfp_gemm_set_epilogue(v)
        res[v].append(t())
L.rrfp_gemm_set_epilogue(1)
for v, name in ((1, "TMA store (local mailbox)"), (2, "staged coalesced st.global (peer mailbox)")):
    us = statistics.median(res[v])
    print(f"fc2 fwd+R 2048x2048x8192, {name:42s}: {us:6.1f} us  {2 * S * D * F / us / 1e6:6.0f} TF/s  "
          f"output {S * D * 2 / 1e6:.1f} MB")
