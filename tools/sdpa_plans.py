"""Enumerate and time the cuDNN SDPA fwd / bwd execution plans for the stage's
attention shape (S=2048, 16 heads x 128, causal) with our strides (dev tool)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cudnn
from paper_2605_18750_b200.attention import _handle
T, H, Dh = 2048, 16, 128
D = H * Dh
dev = torch.device("cuda", 0)
bf, f32 = cudnn.data_type.BFLOAT16, cudnn.data_type.FLOAT
h = _handle(dev)
dim, qs, os_ = [1, H, T, Dh], [T * 3 * D, Dh, 3 * D, 1], [T * D, Dh, D, 1]
sd, ss = [1, H, T, 1], [H * T, T, 1, 1]
qkv = torch.randn(T, 3 * D, device=dev).to(torch.bfloat16)
o = torch.empty(T, D, device=dev, dtype=torch.bfloat16)
st = torch.empty(H, T, device=dev)
do = torch.randn(T, D, device=dev).to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
e = 2 * D


def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for which in ("fwd", "bwd"):
    g = cudnn.pygraph(io_data_type=bf, intermediate_data_type=f32, compute_data_type=f32, handle=h)
    q = g.tensor(name="q", dim=dim, stride=qs, data_type=bf)
    k = g.tensor(name="k", dim=dim, stride=qs, data_type=bf)
    v = g.tensor(name="v", dim=dim, stride=qs, data_type=bf)
    if which == "fwd":
        oo, stt = g.sdpa(name="s", q=q, k=k, v=v, generate_stats=True, attn_scale=1 / math.sqrt(Dh), use_causal_mask=True)
        oo.set_output(True).set_dim(dim).set_stride(os_).set_data_type(bf)
        stt.set_output(True).set_dim(sd).set_stride(ss).set_data_type(f32)
        pack = {q: qkv.data_ptr(), k: qkv.data_ptr() + e, v: qkv.data_ptr() + 2 * e,
                oo: o.data_ptr(), stt: st.data_ptr()}
    else:
        oo = g.tensor(name="o", dim=dim, stride=os_, data_type=bf)
        dd = g.tensor(name="do", dim=dim, stride=os_, data_type=bf)
        stt = g.tensor(name="st", dim=sd, stride=ss, data_type=f32)
        dq, dk, dv = g.sdpa_backward(name="b", q=q, k=k, v=v, o=oo, dO=dd, stats=stt, attn_scale=1 / math.sqrt(Dh),
                                     use_causal_mask=True)
        for t in (dq, dk, dv):
            t.set_output(True).set_dim(dim).set_stride(qs).set_data_type(bf)
        pack = {q: qkv.data_ptr(), k: qkv.data_ptr() + e, v: qkv.data_ptr() + 2 * e,
                oo: o.data_ptr(), dd: do.data_ptr(), stt: st.data_ptr(),
                dq: dqkv.data_ptr(), dk: dqkv.data_ptr() + e, dv: dqkv.data_ptr() + 2 * e}
    g.validate(); g.build_operation_graph()
    g.create_execution_plans([cudnn.heur_mode.A, cudnn.heur_mode.B, cudnn.heur_mode.FALLBACK])
    g.check_support()
    g.build_plans(cudnn.build_plan_policy.ALL)
    n = g.get_execution_plan_count()
    print(which, "plans", n, flush=True)
    for i in range(n):
        try:
            ws = torch.empty(max(g.get_workspace_size_plan_at_index(i), 16), device=dev, dtype=torch.uint8)
            t = timeit(lambda: g.execute_plan_at_index(pack, ws, i, handle=h))
            print(f"  {i}: {g.get_plan_name_at_index(i)[:70]:70s} {t:8.1f} us", flush=True)
        except Exception as ex:
            print(f"  {i}: failed {str(ex)[:100]}", flush=True)
