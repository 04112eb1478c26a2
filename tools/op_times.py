"""Per-op CUDA-event timing of one microbatch's F and B (eager, dev tool)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18750_b200 import kernels as K, model as Mo
from paper_2605_18750_b200.model import GPTConfig, StageCompute

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
st = StageCompute(GPTConfig(n_layer=L), 0, 1, 2, "cuda")
times = collections.defaultdict(list)

def wrap(name, fn):
    def w(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(*a, **k); e1.record()
        times[name].append((e0, e1))
        return r
    return w

def gemm_name(a, b, c, **kw):
    return f"gemm epi{kw.get('epi', 0)} a_mn{int(kw.get('a_mn', False))} b_mn{int(kw.get('b_mn', False))} {tuple(c.shape) if hasattr(c, 'shape') else ''}"

orig_gemm = K.gemm
def g(a, b, c, **kw):
    return wrap(gemm_name(a, b, c, **kw), orig_gemm)(a, b, c, **kw)
K.gemm = g
Mo._ln_fwd = wrap("ln_fwd", Mo._ln_fwd)
Mo._ln_bwd = wrap("ln_bwd", Mo._ln_bwd)
Mo._bias_grad = wrap("bias_grad", Mo._bias_grad)
st._attn_fwd = wrap("attn_fwd(+aux)", st._attn_fwd)
st._attn_bwd = wrap("attn_bwd(+pack)", st._attn_bwd)
st.side = torch.cuda.current_stream()  # serialize for attribution
for it in range(3):
    times.clear()
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(); st.forward(0); b.record(); st.backward_input(0); c.record()
    torch.cuda.synchronize()
print(f"L={L}: F {a.elapsed_time(b):.3f} ms  B {b.elapsed_time(c):.3f} ms (eager, serialized side stream)")
rows = []
for k, v in times.items():
    tot = sum(x.elapsed_time(y) for x, y in v)
    rows.append((tot, len(v), k))
for tot, n, k in sorted(rows, reverse=True):
    print(f"{tot*1e3:9.1f} us  x{n:3d}  {tot*1e3/n:8.1f} us/call  {k}")
