"""Interleaved A/B/C of the stage GEMMs (bench.py's roofline set): full last
wave, half-width tail (rrfp_gemm_set_tail_split), two-pair clusters with A
multicast (rrfp_gemm_set_multicast), and the sub-wave shapes (2048^3) as
halves / stream-K (rrfp_gemm_set_small); 10 alternating rounds of 30 launches
per variant, median per variant (dev tool)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18750_b200 import _lib
from paper_2605_18750_b200.model import GPTConfig

L = _lib.lib()
calls = bench.roofline_gemm_calls(GPTConfig())
names = ["qkv fwd", "proj fwd+R", "fc1 fwd gelu", "fc2 fwd+R", "fc2 dgrad gelu'", "fc1 dgrad", "qkv dgrad",
         "fc2 wgrad f32+=", "fc1 wgrad f32+=", "qkv wgrad f32+=", "proj dgrad", "proj wgrad f32+="]


def t(fn, reps=30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


VARS = [("r-prefetch", 1, 1, 0), ("no-prefetch", 1, 1, 0x100), ("sk-wgrad", 1, 1, 1)]
print(f"co-resident clusters: pairs {L.rrfp_gemm_max_clusters(1)}, two-pair clusters {L.rrfp_gemm_max_clusters(2)}",
      flush=True)


def setv(ts, mc, sm):
    L.rrfp_gemm_set_tail_split(ts)
    L.rrfp_gemm_set_multicast(mc)
    L.rrfp_gemm_set_small(sm & 0xff)
    L.rrfp_gemm_set_rpref(0 if sm & 0x100 else 1)


for _ in range(3):           # warm every shape / variant first (clocks settle under load)
    for fn, _ in calls:
        for _, ts, mc, sm in VARS:
            setv(ts, mc, sm)
            t(fn, 30)
tot = {v[0]: 0.0 for v in VARS}
ftot = 0.0
for (fn, fl), nm in zip(calls, names):
    res = {v[0]: [] for v in VARS}
    for _ in range(10):
        for name, ts, mc, sm in VARS:
            setv(ts, mc, sm)
            res[name].append(t(fn))
    ftot += fl
    line = f"{nm:18s}"
    for name, _, _, _ in VARS:
        m = statistics.median(res[name])
        tot[name] += m
        line += f"  {name} {m:6.1f}us {fl / m / 1e6:5.0f}TF/s"
    print(line, flush=True)
print(f"{'layer':18s}" + "".join(f"  {n} {tot[n]:6.1f}us {ftot / tot[n] / 1e6:5.0f}TF/s" for n, _, _, _ in VARS))
setv(1, 1, 0)
