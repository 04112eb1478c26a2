"""Run one layer's twelve F/B/W stage GEMMs (bench.py's roofline set): 3 warm-up
rounds, then one profiled round (for ncu --set full -k regex:gemm_bf16 -s 36 -c 12)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_18750_b200.model import GPTConfig
calls = bench.roofline_gemm_calls(GPTConfig())
for _ in range(3):
    for c, _ in calls: c()
torch.cuda.synchronize()
for c, _ in calls: c()
torch.cuda.synchronize()
print("done")
