"""Attention core (csrc/fmha_sm100.cu) against a plain PyTorch fp32
reference of the same op on the same packed QKV.

Tolerances: bf16 output O -> max |err| / max |ref| < 2e-2 (P is rounded to bf16
before the PV product, as in every flash kernel); the row statistics lse (fp32,
natural-log logsumexp) -> |err| < 1e-3 * max(1, |ref|)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_fwd(qkv, H, causal, scale):
    T = qkv.shape[0]
    D = H * 128
    q, k, v = (qkv[:, i * D:(i + 1) * D].float().view(T, H, 128).transpose(0, 1) for i in range(3))
    s = (q @ k.transpose(1, 2)) * scale
    if causal:
        s = s.masked_fill(torch.ones(T, T, dtype=torch.bool, device=qkv.device).triu(1), float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    o = torch.softmax(s, dim=-1) @ v
    return o.transpose(0, 1).reshape(T, D), lse


def _qkv(T, H, seed, pad=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    D = H * 128
    x = torch.randn(T, 3 * D + pad, device="cuda", generator=g)
    x[:, :2 * D] *= 1.5   # peaky rows: exercises the lazy rescale
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("T,H,causal", [(128, 1, True), (256, 2, True), (384, 1, True), (2048, 16, True),
                                        (256, 2, False), (384, 3, False), (1024, 4, False)])
def test_attn_fwd_matches_fp32(T, H, causal):
    from paper_2605_18750_b200 import kernels as K
    qkv = _qkv(T, H, T + H)
    D = H * 128
    o = torch.zeros(T, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(H, T, device="cuda")
    K.attn_fwd(qkv, o, lse, heads=H, causal=causal)
    torch.cuda.synchronize()
    want, wl = _ref_fwd(qkv, H, causal, 128 ** -0.5)
    err = (o.float() - want).abs().max().item()
    assert err / want.abs().max().item() < 2e-2, err
    assert ((lse - wl).abs() / wl.abs().clamp(min=1)).max().item() < 1e-3


def test_attn_fwd_strided_views():
    """O written into a wider activation row, lse rows longer than T (stats_row)."""
    from paper_2605_18750_b200 import kernels as K
    T, H = 512, 2
    qkv = _qkv(T, H, 7, pad=64)
    D = H * 128
    obuf = torch.full((T, D + 64), 7.0, device="cuda", dtype=torch.bfloat16)
    lbuf = torch.full((H, T + 128), 7.0, device="cuda")
    K.attn_fwd(qkv, obuf[:, :D], lbuf[:, :T], heads=H, causal=True, T=T)
    torch.cuda.synchronize()
    want, wl = _ref_fwd(qkv, H, True, 128 ** -0.5)
    assert (obuf[:, D:] == 7.0).all() and (lbuf[:, T:] == 7.0).all()
    assert (obuf[:, :D].float() - want).abs().max().item() / want.abs().max().item() < 2e-2
    assert ((lbuf[:, :T] - wl).abs()).max().item() < 1e-2


def test_attn_fwd_stats_match_cudnn():
    """The lse rows are the softmax statistics cuDNN's SDPA writes (same layout),
    so either backward can consume either forward."""
    from paper_2605_18750_b200 import kernels as K
    from paper_2605_18750_b200.attention import sdpa_graphs
    T, H = 2048, 16
    qkv = _qkv(T, H, 11)
    D = H * 128
    o = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, T, device="cuda")
    K.attn_fwd(qkv, o, lse, heads=H, causal=True)
    g = sdpa_graphs(T, H, 128, True, torch.device("cuda"), T)
    ws = torch.empty(max(g.workspace_bytes, 16), device="cuda", dtype=torch.uint8)
    oc = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    st = torch.empty(H, T, device="cuda")
    g.forward(qkv.data_ptr(), oc.data_ptr(), st.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (lse - st).abs().max().item() < 1e-2
    assert (o.float() - oc.float()).abs().max().item() < 3e-2


def _ref_bwd(qkv, do, H, causal, scale):
    T = qkv.shape[0]
    D = H * 128
    x = qkv.float().requires_grad_(True)
    q, k, v = (x[:, i * D:(i + 1) * D].view(T, H, 128).transpose(0, 1) for i in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal, scale=scale)
    o = o.transpose(0, 1).reshape(T, D)
    o.backward(do.float())
    return x.grad


@pytest.mark.parametrize("T,H,causal", [(128, 1, True), (256, 2, True), (384, 1, True), (2048, 16, True),
                                        (256, 2, False), (384, 3, False)])
def test_attn_bwd_matches_fp32(T, H, causal):
    """dQ, dK, dV (packed) against fp32 autograd: per block cosine >= 0.999, relative L2 <= 2e-2."""
    from paper_2605_18750_b200 import kernels as K
    qkv = _qkv(T, H, 3 * T + H)
    D = H * 128
    g = torch.Generator(device="cuda").manual_seed(T + 5)
    do = torch.randn(T, D, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.zeros(T, D, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(H, T, device="cuda")
    K.attn_fwd(qkv, o, lse, heads=H, causal=causal)
    dqkv = torch.full((T, 3 * D), 7.0, device="cuda", dtype=torch.bfloat16)
    ws = K.attn_bwd_workspace(T, H)
    K.attn_bwd(qkv, o, do, lse, dqkv, ws, heads=H, causal=causal)
    torch.cuda.synchronize()
    want = _ref_bwd(qkv, do, H, causal, 128 ** -0.5)
    for i, name in enumerate("qkv"):
        a, b = dqkv[:, i * D:(i + 1) * D].float(), want[:, i * D:(i + 1) * D]
        cos = torch.nn.functional.cosine_similarity(a.flatten(), b.flatten(), dim=0).item()
        rel = ((a - b).norm() / b.norm()).item()
        assert cos >= 0.999 and rel <= 2e-2, (name, cos, rel)
