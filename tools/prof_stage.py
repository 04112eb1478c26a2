"""Profile one microbatch's F + B of a GPT-1.3B stage (L layers), eager (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200.model import GPTConfig, StageCompute
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dec = len(sys.argv) > 2 and sys.argv[2] == "bfw"
st = StageCompute(GPTConfig(n_layer=L), 0, 1, 1, "cuda", decompose=dec)
for i in range(3):
    st.forward(0); st.backward_input(0)
    if dec: st.backward_weight(0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.forward(0); st.backward_input(0)
if dec: st.backward_weight(0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
