"""Captured F / B / W task-body times of a GPT-1.3B stage (CUDA graphs replayed
back to back, CUDA events), comparing B-task stream layouts (dev tool).
    python tools/task_times.py [layers] [bfw]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200.model import GPTConfig, StageCompute

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dec = len(sys.argv) > 2 and sys.argv[2] == "bfw"


def run(single_stream, label):
    st = StageCompute(GPTConfig(n_layer=L), 1, 3, 2, "cuda", decompose=dec)   # interior stage
    if single_stream:
        st.side = None
    st.capture_bodies()
    kinds = ["F", "B"] + (["W"] if dec else [])
    res = {}
    for k in kinds:
        g = st.graphs[(k, 0)]
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[k] = e0.elapsed_time(e1) / 10 * 1e3 / len(st.layers)
    print(f"{label:28s} " + "  ".join(f"{k} {v:7.1f} us/layer" for k, v in res.items()), flush=True)
    del st
    torch.cuda.empty_cache()


run(False, "B on two streams")
run(True, "B on one stream")
