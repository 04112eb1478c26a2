"""One interior-stage layer's captured F and B bodies replayed (for an ncu launch
list with --cache-control none: warm-L2 per-kernel times inside the task graphs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200.model import GPTConfig, StageCompute
st = StageCompute(GPTConfig(n_layer=3), 1, 3, 2, "cuda")   # one layer, interior stage
st.capture_bodies()
for _ in range(3):
    st.graphs[("F", 0)].replay(); st.graphs[("B", 0)].replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.graphs[("F", 1)].replay(); st.graphs[("B", 1)].replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
