"""Do green-context SM partitions confine (a) eager kernels, (b) CUDA graphs
captured on a green stream and replayed elsewhere, (c) those graphs as child
nodes of another graph?  (dev probe for the PP emulation)"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import _lib, kernels as K
L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
arr = (C.c_void_p * (2 * n))()
sms = C.c_int()
rc = L.rrfp_green_streams(0, n, 148 // n // 2 * 2 - 2, arr, C.byref(sms))
print("green rc", rc, L.rrfp_last_error(), "sms/part", sms.value, flush=True)
if rc:
    sys.exit(0)
gs = torch.cuda.ExternalStream(arr[0])
x = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
w = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
y = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
torch.cuda.synchronize()

def t(fn, stream, reps=5):
    with torch.cuda.stream(stream):
        fn()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        for _ in range(reps): fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

ns = torch.cuda.Stream()
cap = sms.value
print("eager full GPU", round(t(lambda: K.gemm(x, w, y), ns), 3), "ms", flush=True)
L.rrfp_gemm_reserve_sms(148 - cap)
print("eager capped grid, normal stream", round(t(lambda: K.gemm(x, w, y), ns), 3), "ms", flush=True)
L.rrfp_gemm_reserve_sms(0)
print("eager full grid, green stream", round(t(lambda: K.gemm(x, w, y), gs), 3), "ms", flush=True)
g = torch.cuda.CUDAGraph(keep_graph=True)
with torch.cuda.graph(g, stream=gs):
    K.gemm(x, w, y)
g.instantiate() if hasattr(g, "instantiate") else None
print("graph captured on green, replayed on normal stream", round(t(lambda: g.replay(), ns), 3), "ms", flush=True)
print("torch matmul on green stream", round(t(lambda: torch.matmul(x, w, out=y), gs), 3), "ms", flush=True)
