"""HBM-bound stage kernels (csrc/ops.cu) against plain PyTorch fp32 references.

Tolerances: bf16 outputs -> max |err| / max |ref| < 1e-2; fp32 statistics
(loss, lse, LayerNorm parameter gradients) -> rtol 1e-3."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def _L():
    from paper_2605_18750_b200 import _lib
    return _lib.lib()


def _p(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _close(got, want, tol=1e-2):
    err = (got.float() - want.float()).abs().max().item()
    assert err / (want.float().abs().max().item() + 1e-6) < tol, err


@pytest.mark.parametrize("rows,V", [(64, 50304), (7, 1000), (3, 8)])
def test_xent_fwd_bwd(rows, V):
    torch.manual_seed(rows)
    logits = (torch.randn(rows, V, device="cuda") * 3).to(torch.bfloat16)
    tgt = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    loss = torch.zeros(rows, device="cuda")
    lse = torch.zeros(rows, device="cuda")
    assert _L().rrfp_xent_fwd(_p(logits), C.c_longlong(V), _p(tgt), rows, V, _p(loss), _p(lse), _st()) == 0
    torch.cuda.synchronize()
    lf = logits.float()
    want_lse = torch.logsumexp(lf, dim=1)
    torch.testing.assert_close(lse, want_lse, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(loss, want_lse - lf[torch.arange(rows), tgt.long()], rtol=1e-4, atol=1e-4)
    scale = 0.5
    assert _L().rrfp_xent_bwd(_p(logits), C.c_longlong(V), _p(tgt), rows, V, _p(lse), C.c_float(scale), _st()) == 0
    torch.cuda.synchronize()
    want = (torch.softmax(lf, 1) - torch.nn.functional.one_hot(tgt.long(), V)) * scale
    _close(logits, want)


@pytest.mark.parametrize("rows,D", [(256, 2048), (100, 1280), (64, 4096), (33, 256)])
def test_layernorm_fwd_bwd(rows, D):
    torch.manual_seed(D)
    bf = torch.bfloat16
    x = torch.randn(rows, D, device="cuda").to(bf)
    g = (1 + 0.1 * torch.randn(D, device="cuda")).to(bf)
    b = (0.1 * torch.randn(D, device="cuda")).to(bf)
    y = torch.empty_like(x)
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    assert _L().rrfp_layernorm_fwd(_p(x), _p(g), _p(b), _p(y), _p(mean), _p(rstd), rows, D,
                                   C.c_float(1e-5), _st()) == 0
    xr = x.float().requires_grad_(True)
    gr, br = g.float().requires_grad_(True), b.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (D,), gr, br, 1e-5)
    torch.cuda.synchronize()
    _close(y, yr)
    dy = torch.randn(rows, D, device="cuda").to(bf)
    dres = torch.randn(rows, D, device="cuda").to(bf)
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    dg, db = torch.zeros(D, device="cuda"), torch.zeros(D, device="cuda")
    assert _L().rrfp_layernorm_bwd(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), _p(dres), _p(dx), _p(dg),
                                   _p(db), rows, D, _st()) == 0
    torch.cuda.synchronize()
    _close(dx, xr.grad + dres.float())
    torch.testing.assert_close(dg, gr.grad, rtol=1e-3, atol=1e-3)
    torch.testing.assert_close(db, br.grad, rtol=1e-3, atol=1e-3)
    # parameter gradients only (dx = NULL) accumulate on top
    assert _L().rrfp_layernorm_bwd(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), None, None, _p(dg),
                                   _p(db), rows, D, _st()) == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(db, 2 * br.grad, rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("rows,D", [(2048, 2048), (100, 1280), (2048, 4096), (33, 256), (3, 512)])
def test_layernorm_bwd_fused(rows, D):
    """One-pass LN backward: dx (+ dres), dg / db and the column sums of dres and
    dx (adjacent bias gradients), each accumulated; every output optional."""
    torch.manual_seed(D + rows)
    bf = torch.bfloat16
    x = torch.randn(rows, D, device="cuda").to(bf)
    g = (1 + 0.1 * torch.randn(D, device="cuda")).to(bf)
    mean = x.float().mean(1)
    rstd = torch.rsqrt(x.float().var(1, unbiased=False) + 1e-5)
    xr = x.float().requires_grad_(True)
    gr = g.float().requires_grad_(True)
    br = torch.zeros(D, device="cuda", requires_grad=True)
    yr = torch.nn.functional.layer_norm(xr, (D,), gr, br, 1e-5)
    dy = torch.randn(rows, D, device="cuda").to(bf)
    dres = torch.randn(rows, D, device="cuda").to(bf)
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    base = torch.randn(4, D, device="cuda")
    dg, db, cr, cd = (base[i].clone() for i in range(4))
    assert _L().rrfp_layernorm_bwd_fused(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), _p(dres), _p(dx), _p(dg),
                                         _p(db), _p(cr), _p(cd), rows, D, _st()) == 0
    torch.cuda.synchronize()
    want_dx = xr.grad + dres.float()
    _close(dx, want_dx)
    torch.testing.assert_close(dg, base[0] + gr.grad, rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(db, base[1] + br.grad, rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(cr, base[2] + dres.float().sum(0), rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(cd, base[3] + want_dx.sum(0), rtol=1e-3, atol=0.05)
    # reductions only: no dx, dres feeds only its column sum
    dg2, cr2 = torch.zeros(D, device="cuda"), torch.zeros(D, device="cuda")
    assert _L().rrfp_layernorm_bwd_fused(_p(dy), _p(x), _p(mean), _p(rstd), None, _p(dres), None, _p(dg2),
                                         None, _p(cr2), None, rows, D, _st()) == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(dg2, gr.grad, rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(cr2, dres.float().sum(0), rtol=1e-3, atol=2e-3)
    # argument checks: cs_dx without dx, width > 4096
    assert _L().rrfp_layernorm_bwd_fused(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), None, None, None,
                                         None, None, _p(cd), rows, D, _st()) != 0
    assert _L().rrfp_layernorm_bwd_fused(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), None, _p(dx), None,
                                         None, None, None, 1, 8192, _st()) != 0


def test_layernorm_rejects_bad_width():
    x = torch.zeros(4, 300, device="cuda", dtype=torch.bfloat16)
    assert _L().rrfp_layernorm_fwd(_p(x), _p(x), _p(x), _p(x), _p(x), _p(x), 4, 300, C.c_float(1e-5), _st()) != 0


@pytest.mark.parametrize("rows,cols", [(2048, 2048), (100, 1024)])
def test_bias_grad_colsum(rows, cols):
    torch.manual_seed(cols)
    dy = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    db = torch.ones(cols, device="cuda")
    assert _L().rrfp_bias_grad(_p(dy), C.c_longlong(cols), _p(db), rows, cols, _st()) == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(db, 1 + dy.float().sum(0), rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("rows,D,V", [(256, 2048, 64), (100, 1280, 7), (2048, 2048, 50304)])
def test_embedding_fwd_bwd(rows, D, V):
    """x = E[tok] + P[pos]; backward scatter-adds into E (tokens repeat: V small
    forces collisions) and adds into P, on top of existing gradient values."""
    g = torch.Generator(device="cuda").manual_seed(rows)
    tok = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32, generator=g)
    E = torch.randn(V, D, device="cuda", generator=g).bfloat16()
    P = torch.randn(rows, D, device="cuda", generator=g).bfloat16()
    x = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
    L = _L()
    assert L.rrfp_embedding_fwd(_p(tok), _p(E), _p(P), _p(x), rows, D, _st()) == 0
    dx = torch.randn(rows, D, device="cuda", generator=g).bfloat16()
    dE = torch.randn(V, D, device="cuda", generator=g)
    dP = torch.randn(rows, D, device="cuda", generator=g)
    wantE = dE.clone().index_add_(0, tok.long(), dx.float())
    wantP = dP + dx.float()
    assert L.rrfp_embedding_bwd(_p(tok), _p(dx), _p(dE), _p(dP), rows, D, _st()) == 0
    torch.cuda.synchronize()
    _close(x, E.float()[tok.long()] + P.float())
    torch.testing.assert_close(dE, wantE, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(dP, wantP, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("rows,D,V", [(2048, 2048, 50304), (256, 256, 1000), (200, 512, 4096)])
def test_lm_head_xent_fused(rows, D, V):
    """LM head GEMM with the softmax-statistics epilogue + xent_combine against
    GEMM + xent_fwd (same bf16 logits, bit-identical) and an fp32 reference."""
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(V)
    bf = torch.bfloat16
    hf = torch.randn(rows, D, device="cuda").to(bf)
    w = (torch.randn(V, D, device="cuda") * 0.05).to(bf)
    tgt = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    logits = torch.empty(rows, V, device="cuda", dtype=bf)
    loss, lse = torch.zeros(rows, device="cuda"), torch.zeros(rows, device="cuda")
    part = torch.full((rows, Kn.lm_head_slots(V), 2), float("nan"), device="cuda")
    Kn.lm_head_xent_fwd(hf, w, logits, tgt, loss, lse, part)
    ref_logits = torch.empty_like(logits)
    Kn.gemm(hf, w, ref_logits)
    loss2, lse2 = torch.zeros(rows, device="cuda"), torch.zeros(rows, device="cuda")
    assert _L().rrfp_xent_fwd(_p(ref_logits), C.c_longlong(V), _p(tgt), rows, V, _p(loss2), _p(lse2), _st()) == 0
    torch.cuda.synchronize()
    assert torch.equal(logits, ref_logits)
    torch.testing.assert_close(lse, lse2, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(loss, loss2, rtol=1e-5, atol=1e-4)
    lf = logits.float()
    want = torch.logsumexp(lf, 1)
    torch.testing.assert_close(lse, want, rtol=1e-5, atol=1e-4)
    torch.testing.assert_close(loss, want - lf[torch.arange(rows), tgt.long()], rtol=1e-5, atol=1e-4)
