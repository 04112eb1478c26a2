"""Interleaved A/B of the stage GEMMs (bench.py's roofline set): full last wave
vs half-width tail (rrfp_gemm_set_tail_split), 6 alternating rounds of 30
launches per variant, median per variant (dev tool)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18750_b200 import _lib
from paper_2605_18750_b200.model import GPTConfig

L = _lib.lib()
calls = bench.roofline_gemm_calls(GPTConfig())
names = ["qkv fwd", "proj fwd+R", "fc1 fwd gelu", "fc2 fwd+R", "fc2 dgrad gelu'", "fc1 dgrad", "qkv dgrad",
         "fc2 wgrad f32+=", "fc1 wgrad f32+=", "qkv wgrad f32+="]


def t(fn, reps=30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for fn, _ in calls:          # warm every shape / variant first
    for ts in (0, 1):
        L.rrfp_gemm_set_tail_split(ts)
        t(fn, 10)
tot = {0: 0.0, 1: 0.0}
ftot = 0.0
for (fn, fl), nm in zip(calls, names):
    res = {0: [], 1: []}
    for _ in range(6):
        for ts in (0, 1):
            L.rrfp_gemm_set_tail_split(ts)
            res[ts].append(t(fn))
    m = {ts: statistics.median(v) for ts, v in res.items()}
    tot[0] += m[0]; tot[1] += m[1]; ftot += fl
    print(f"{nm:18s} full wave {m[0]:6.1f}us {fl / m[0] / 1e6:5.0f}TF/s   half tail {m[1]:6.1f}us "
          f"{fl / m[1] / 1e6:5.0f}TF/s   {100 * (m[0] / m[1] - 1):+.1f}%", flush=True)
print(f"{'layer':18s} full wave {tot[0]:6.1f}us {ftot / tot[0] / 1e6:5.0f}TF/s   half tail {tot[1]:6.1f}us "
      f"{ftot / tot[1] / 1e6:5.0f}TF/s   {100 * (tot[0] / tot[1] - 1):+.1f}%")
L.rrfp_gemm_set_tail_split(1)
