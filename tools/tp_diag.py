"""TP=2 pipeline bring-up diagnostics (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200.model import GPTConfig
from paper_2605_18750_b200.pipeline import GpuPipeline
cfg = GPTConfig(n_layer=4, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=256)
t0 = time.time()
pipe = GpuPipeline(cfg, int(sys.argv[1]) if len(sys.argv) > 1 else 1, 4, tp_size=2)
print("built", round(time.time() - t0, 2), "s; errors", [st.tp.error() for row in pipe.grid for st in row], flush=True)
for i in range(3):
    t0 = time.time()
    loss = pipe.step(watchdog_secs=60).item()
    print("step", i, round(time.time() - t0, 3), "s loss", loss, "errors", [st.tp.error() for row in pipe.grid for st in row], flush=True)
pipe.close()
