"""tcgen05/TMA GEMM numerics against a torch fp32 reference of the same op."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[(1, 1, 64, 0, 1, 3), (1, 1, 128, 0, 1, 3), (1, 2, 64, 0, 1, 3), (1, 0, 64, 0, 1, 3),
                        (0, 0, 64, 0, 1, 3), (1, 1, 64, 1, 1, 3), (1, 2, 64, 1, 1, 3), (1, 1, 64, 0, 0, 3),
                        (1, 1, 64, 1, 1, 0), (1, 2, 64, 1, 1, 0)],   # (small = 3: the measured-slower modes, kept tested)
                # (pair, epilogue, bk, multicast, tail, small: sub-wave shapes as halves / stream-K)
                ids=["pair-tma-store", "pair-bk128", "pair-staged-coalesced", "pair-st-global", "single",
                     "pair-multicast", "pair-multicast-coalesced", "pair-full-last-wave",
                     "pair-multicast-default", "pair-multicast-coalesced-default"],
                autouse=True)
def variant(request):
    from paper_2605_18750_b200 import _lib
    pair, tma, bk, mc, tail, small = request.param
    L = _lib.lib()
    L.rrfp_gemm_set_variant(pair)
    L.rrfp_gemm_set_epilogue(tma)
    L.rrfp_gemm_set_bk(bk)
    L.rrfp_gemm_set_multicast(mc)
    L.rrfp_gemm_set_tail_split(tail)
    L.rrfp_gemm_set_small(small)
    yield request.param
    L.rrfp_gemm_set_variant(1)
    L.rrfp_gemm_set_epilogue(1)
    L.rrfp_gemm_set_bk(64)
    L.rrfp_gemm_set_multicast(1)
    L.rrfp_gemm_set_tail_split(1)
    L.rrfp_gemm_set_small(0)


def _rand(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def _close(got, want, tol=2e-2):
    err = (got.float() - want).abs().max().item()
    ref = want.abs().max().item() + 1e-6
    assert err / ref < tol, (err, ref)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (2048, 6144, 2048),
                                   (384, 300, 192), (200, 256, 128), (200, 320, 128),
                                   (2048, 50304, 2048)])
def test_gemm_forward_kk(M, N, K):
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(0)
    a, b = _rand(M, K), _rand(N, K)
    bias = _rand(N)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    Kn.gemm(a, b, c, bias=bias)
    torch.cuda.synchronize()
    _close(c, a.float() @ b.float().t() + bias.float())


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (2048, 2048, 8192)])
def test_gemm_dgrad_kmn(M, N, K):
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(1)
    dy, w = _rand(M, K), _rand(K, N)       # dX[M,N] = dY[M,K] . W[K,N]
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    Kn.gemm(dy, w, c, b_mn=True)
    torch.cuda.synchronize()
    _close(c, dy.float() @ w.float())


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (200, 320, 128), (6144, 2048, 2048)])
def test_gemm_wgrad_mnmn_accumulate(M, N, K):
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(2)
    dy, x = _rand(K, M), _rand(K, N)       # dW[M,N] += dY^T . X, contraction over K tokens
    acc = torch.randn(M, N, device="cuda")
    want = acc + dy.float().t() @ x.float()
    Kn.gemm(dy, x, acc, epi=Kn.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True)
    torch.cuda.synchronize()
    _close(acc, want, 1e-2)


def test_gemm_fused_epilogues():
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(3)
    M, N, K = 256, 512, 256
    a, b, bias, res = _rand(M, K), _rand(N, K), _rand(N), _rand(M, N)
    ref = a.float() @ b.float().t() + bias.float()
    pre = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(pre)
    Kn.gemm(a, b, pre, epi=Kn.EPI_BIAS_GELU, c2=act, bias=bias)
    out = torch.empty_like(pre)
    Kn.gemm(a, b, out, epi=Kn.EPI_RESID, bias=bias, r=res)
    gb = torch.empty_like(pre)
    Kn.gemm(a, b, gb, epi=Kn.EPI_GELU_BWD, r=res)
    torch.cuda.synchronize()
    _close(pre, ref)
    _close(act, torch.nn.functional.gelu(ref, approximate="tanh"))
    _close(out, ref + res.float())
    x = res.float()
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    g = 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)
    _close(gb, (a.float() @ b.float().t()) * g)


@pytest.mark.parametrize("M,N,K", [(256, 512, 128), (200, 320, 64)])
def test_gemm_f32_store(M, N, K):
    """EPI_F32 and EPI_ACC_F32 with accumulate=0 overwrite C (no reduction)."""
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(4)
    a, b = _rand(M, K), _rand(N, K)
    want = a.float() @ b.float().t()
    for epi in (Kn.EPI_F32, Kn.EPI_ACC_F32):
        c = torch.full((M, N), 7.0, device="cuda")
        Kn.gemm(a, b, c, epi=epi, accumulate=False)
        torch.cuda.synchronize()
        _close(c, want, 1e-2)


def test_gemm_fused_epilogues_tails():
    """Row and column tails (M=200, N=320: a partial 256x256 pair tile) for every bf16 epilogue."""
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(5)
    M, N, K = 200, 320, 192
    a, b, bias, res = _rand(M, K), _rand(N, K), _rand(N), _rand(M, N)
    ref = a.float() @ b.float().t() + bias.float()
    pre = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    act = torch.zeros_like(pre)
    Kn.gemm(a, b, pre, epi=Kn.EPI_BIAS_GELU, c2=act, bias=bias)
    out = torch.zeros_like(pre)
    Kn.gemm(a, b, out, epi=Kn.EPI_RESID, bias=bias, r=res)
    torch.cuda.synchronize()
    _close(pre, ref)
    _close(act, torch.nn.functional.gelu(ref, approximate="tanh"))
    _close(out, ref + res.float())


@pytest.mark.parametrize("pairs", [3, 5, 7])
def test_gemm_streamk_fixup_all_epilogues(pairs, variant):
    """Few CTA pairs (SMs reserved) so the last partial round is split over
    clusters with 2-3 contributors per tile: owner fix-up for every epilogue,
    direct reduce-add for the f32 accumulate."""
    from paper_2605_18750_b200 import kernels as Kn, _lib
    if variant[0] == 0:
        pytest.skip("stream-K is a pair-kernel schedule")
    L = _lib.lib()
    n_sms = torch.cuda.get_device_properties(0).multi_processor_count
    L.rrfp_gemm_reserve_sms(n_sms - 2 * pairs)
    L.rrfp_gemm_set_streamk(1)
    try:
        torch.manual_seed(6 + pairs)
        M, N, K = 512, 1024, 960          # 8 tiles of 256x256, 15 k-blocks
        a, b, bias, res = _rand(M, K), _rand(N, K), _rand(N), _rand(M, N)
        ref = a.float() @ b.float().t()
        for _ in range(2):                 # second launch reuses the (self-reset) counters
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            Kn.gemm(a, b, c, bias=bias)
            pre, act = torch.empty_like(c), torch.empty_like(c)
            Kn.gemm(a, b, pre, epi=Kn.EPI_BIAS_GELU, c2=act, bias=bias)
            out = torch.empty_like(c)
            Kn.gemm(a, b, out, epi=Kn.EPI_RESID, bias=bias, r=res)
            gb = torch.empty_like(c)
            Kn.gemm(a, b, gb, epi=Kn.EPI_GELU_BWD, r=res)
            f = torch.full((M, N), 3.0, device="cuda")
            Kn.gemm(a, b, f, epi=Kn.EPI_F32)
            acc = torch.randn(M, N, device="cuda")
            want_acc = acc + ref
            Kn.gemm(a, b, acc, epi=Kn.EPI_ACC_F32, accumulate=True)
            torch.cuda.synchronize()
            _close(c, ref + bias.float())
            _close(pre, ref + bias.float())
            _close(act, torch.nn.functional.gelu(ref + bias.float(), approximate="tanh"))
            _close(out, ref + bias.float() + res.float())
            x = res.float()
            t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
            gg = 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)
            _close(gb, ref * gg)
            _close(f, ref, 1e-2)
            _close(acc, want_acc, 1e-2)
    finally:
        L.rrfp_gemm_reserve_sms(0)
        L.rrfp_gemm_set_streamk(0)


def test_gemm_out_projection_2048_cube():
    """The three 2048^3 GEMMs of the attention out-projection (64 tiles: less
    than one wave of CTA pairs): forward + bias + residual, dgrad, wgrad +=."""
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(7)
    S = D = 2048
    x, w, bias, res = _rand(S, D), _rand(D, D, scale=0.05), _rand(D), _rand(S, D)
    y = torch.empty(S, D, device="cuda", dtype=torch.bfloat16)
    Kn.gemm(x, w, y, epi=Kn.EPI_RESID, bias=bias, r=res)
    dy = _rand(S, D)
    dx = torch.empty(S, D, device="cuda", dtype=torch.bfloat16)
    Kn.gemm(dy, w, dx, b_mn=True)
    gw = torch.randn(D, D, device="cuda")
    want_gw = gw + dy.float().t() @ x.float()
    Kn.gemm(dy, x, gw, epi=Kn.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True)
    torch.cuda.synchronize()
    _close(y, x.float() @ w.float().t() + bias.float() + res.float())
    _close(dx, dy.float() @ w.float())
    _close(gw, want_gw, 1e-2)


@pytest.mark.parametrize("M,N,K", [(2048, 8192, 2048), (200, 320, 192), (256, 512, 256)])
def test_gemm_gelu_bwd_column_sums(M, N, K, variant):
    """EPI_GELU_BWD with C2: the epilogue also accumulates the column sums of
    the stored bf16 output (the FC1 bias gradient) into an fp32 vector (staged
    epilogues only; the per-thread-store variants refuse it)."""
    from paper_2605_18750_b200 import kernels as Kn
    torch.manual_seed(11)
    a, b, pre = _rand(M, K), _rand(N, K), _rand(M, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.randn(N, device="cuda")
    base = cs.clone()
    pair, tma = variant[0], variant[1]
    if not pair or not tma:
        with pytest.raises(RuntimeError):
            Kn.gemm(a, b, out, epi=Kn.EPI_GELU_BWD, r=pre, c2=cs)
        return
    Kn.gemm(a, b, out, epi=Kn.EPI_GELU_BWD, r=pre, c2=cs)
    torch.cuda.synchronize()
    want = base + out.float().sum(0)
    torch.testing.assert_close(cs, want, rtol=1e-4, atol=1e-2)
