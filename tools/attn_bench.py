"""Attention core timing on the GPT-1.3B shape (T=2048, H=16, d_head=128, causal):
csrc/fmha_sm100.cu vs the cuDNN SDPA graph (attention.py), CUDA events on the
launch stream, 20 back-to-back launches after 5 warm-ups (inputs 24 MB: L2
resident, as in the step where the QKV GEMM just wrote them).

    python tools/attn_bench.py [--T 2048] [--H 16] [--bwd]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch


def timeit(fn, reps=200, warm=2000):
    # ~50-100 ms of warm-up so the SM clock has left its idle state
    for _ in range(warm):
        fn()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--H", type=int, default=16)
    ap.add_argument("--noncausal", action="store_true")
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--only-ours", action="store_true")
    a = ap.parse_args()
    from paper_2605_18750_b200 import kernels as K
    T, H = a.T, a.H
    causal = not a.noncausal
    D = H * 128
    qkv = torch.randn(T, 3 * D, device="cuda").to(torch.bfloat16)
    o = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, T, device="cuda")
    flops_f = 4 * T * T * 128 * H / (2 if causal else 1)
    res = {"T": T, "H": H, "causal": causal, "fwd_gflop": flops_f / 1e9}
    us = timeit(lambda: K.attn_fwd(qkv, o, lse, heads=H, causal=causal))
    res["ours_fwd_us"] = round(us, 2)
    res["ours_fwd_tflops"] = round(flops_f / us / 1e6, 1)
    if a.bwd and hasattr(K, "attn_bwd"):
        do = torch.randn(T, D, device="cuda").to(torch.bfloat16)
        dqkv = torch.empty(T, 3 * D, device="cuda", dtype=torch.bfloat16)
        ws2 = K.attn_bwd_workspace(T, H)
        flops_b = 2.5 * flops_f
        us = timeit(lambda: K.attn_bwd(qkv, o, do, lse, dqkv, ws2, heads=H, causal=causal))
        res["ours_bwd_us"] = round(us, 2)
        res["ours_bwd_tflops"] = round(flops_b / us / 1e6, 1)
    if not a.only_ours:
        from paper_2605_18750_b200.attention import sdpa_graphs
        g = sdpa_graphs(T, H, 128, causal, torch.device("cuda"), T)
        ws = torch.empty(max(g.workspace_bytes, 16), device="cuda", dtype=torch.uint8)
        oc = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
        st = torch.empty(H, T, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        us = timeit(lambda: g.forward(qkv.data_ptr(), oc.data_ptr(), st.data_ptr(), ws.data_ptr(), s))
        res["cudnn_fwd_us"] = round(us, 2)
        res["cudnn_fwd_tflops"] = round(flops_f / us / 1e6, 1)
        res["max_abs_diff_vs_cudnn"] = (o.float() - oc.float()).abs().max().item()
        if a.bwd:
            do = torch.randn(T, D, device="cuda").to(torch.bfloat16)
            dq2 = torch.empty(T, 3 * D, device="cuda", dtype=torch.bfloat16)
            us = timeit(lambda: g.backward(qkv.data_ptr(), oc.data_ptr(), do.data_ptr(), st.data_ptr(),
                                           dq2.data_ptr(), ws.data_ptr(), s))
            res["cudnn_bwd_us"] = round(us, 2)
            res["cudnn_bwd_tflops"] = round(2.5 * flops_f / us / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
