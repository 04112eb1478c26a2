"""A/B timing of the ten stage GEMMs of one layer (bench.py's roofline set) under
GEMM variants: CUDA events on one stream, 20 reps after warm-up (dev tool).
    python tools/gemm_ab.py            -> TMA-store epilogue vs per-thread stores
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18750_b200 import _lib
from paper_2605_18750_b200.model import GPTConfig

names = ["qkv fwd", "proj fwd+R", "fc1 fwd gelu", "fc2 fwd+R", "fc2 dgrad gelu'", "fc1 dgrad", "qkv dgrad",
         "fc2 wgrad f32+=", "fc1 wgrad f32+=", "qkv wgrad f32+="]
calls = bench.roofline_gemm_calls(GPTConfig())
L = _lib.lib()
def setv(tma, sk, bk=64):
    return lambda: (L.rrfp_gemm_set_epilogue(tma), L.rrfp_gemm_set_streamk(sk), L.rrfp_gemm_set_bk(bk))
variants = [("bk64 (6 stages)", setv(1, 0, 64)), ("bk128 (3 stages)", setv(1, 0, 128))]
res = {}
for vname, setv in variants:
    setv()
    for (fn, fl), nm in zip(calls, names):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        res[(vname, nm)] = (us, fl / us / 1e6)
hdr = "".join(f"{v:>22s}" for v, _ in variants)
print(f"{'gemm':18s}{hdr}")
tot = {v: 0.0 for v, _ in variants}
for nm in names:
    row = ""
    for v, _ in variants:
        us, tf = res[(v, nm)]
        tot[v] += us
        row += f"{us:10.1f}us {tf:6.0f}TF/s"
    print(f"{nm:18s}{row}")
fl = sum(f for _, f in calls)
print(f"{'layer total':18s}" + "".join(f"{tot[v]:10.1f}us {fl / tot[v] / 1e6:6.0f}TF/s" for v, _ in variants))
