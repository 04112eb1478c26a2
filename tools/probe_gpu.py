"""One-off GPU probe: attention backends and GEMM throughput (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

q = torch.randn(1, 16, 2048, 128, device="cuda", dtype=torch.bfloat16, requires_grad=True)
k = torch.randn_like(q, requires_grad=True); v = torch.randn_like(q, requires_grad=True)
from torch.nn.attention import sdpa_kernel, SDPBackend
for be in (SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    try:
        with sdpa_kernel(be):
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            g = torch.randn_like(o)
            tf = bench(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))
            def fb():
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True); o.backward(g)
            tfb = bench(fb)
        fl = 4 * 2048 * 2048 * 128 * 16 / 2
        print(f"{be}: fwd {tf*1e3:.1f}us ({fl/tf/1e9:.0f} TF/s) fwd+bwd {tfb*1e3:.1f}us", flush=True)
    except Exception as ex:
        print(f"{be}: FAILED {type(ex).__name__}: {str(ex)[:200]}", flush=True)
try:
    import flash_attn
    from flash_attn import flash_attn_func
    qq = q.detach().transpose(1, 2).contiguous(); kk = k.detach().transpose(1, 2).contiguous(); vv = v.detach().transpose(1,2).contiguous()
    tf = bench(lambda: flash_attn_func(qq, kk, vv, causal=True))
    print(f"flash_attn {flash_attn.__version__}: fwd {tf*1e3:.1f}us", flush=True)
except Exception as ex:
    print("flash_attn FAILED", type(ex).__name__, str(ex)[:200], flush=True)

from paper_2605_18750_b200 import kernels as Kn, _lib
_lib.lib().rrfp_gemm_set_epilogue(int(os.environ.get("RRFP_GEMM_TMA_STORE", "1")))
for (M, N, K, am, bm, name) in [(2048, 6144, 2048, 0, 0, "qkv fwd"), (2048, 8192, 2048, 0, 0, "fc1 fwd"),
                                (2048, 2048, 8192, 0, 0, "fc2 fwd"), (2048, 2048, 2048, 0, 0, "proj fwd"),
                                (2048, 2048, 8192, 0, 1, "fc1 dgrad"), (8192, 2048, 2048, 1, 1, "fc1 wgrad"),
                                (2048, 50304, 2048, 0, 0, "lmhead fwd"), (8192, 8192, 8192, 0, 0, "8k^3")]:
    a = torch.randn((K, M) if am else (M, K), device="cuda").to(torch.bfloat16)
    b = torch.randn((K, N) if bm else (N, K), device="cuda").to(torch.bfloat16)
    if am:
        c = torch.zeros(M, N, device="cuda")
        fn = lambda: Kn.gemm(a, b, c, epi=Kn.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True)
    else:
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fn = lambda: Kn.gemm(a, b, c, b_mn=bool(bm))
    t = bench(fn)
    ta = torch.randn(M, K, device="cuda").to(torch.bfloat16); tb = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    tt = bench(lambda: ta @ tb)
    print(f"gemm {name} {M}x{N}x{K}: ours {t*1e3:.1f}us {2*M*N*K/t/1e9:.0f} TF/s | cublas {tt*1e3:.1f}us {2*M*N*K/tt/1e9:.0f} TF/s", flush=True)
