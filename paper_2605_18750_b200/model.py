"""Synthetic GPT stage compute: the F / B / W task bodies.

A ``StageCompute`` owns one pipeline stage's slice of a GPT stack (embedding
on stage 0, LM head + softmax cross-entropy on the last stage), its bf16
weights, fp32 gradient accumulators, per-microbatch activation slots and the
mailbox buffers its neighbours write into.  ``forward(mb)``,
``backward_input(mb)`` and ``backward_weight(mb)`` enqueue the task's kernels
on the current stream; ``capture_bodies()`` records one CUDA graph per
(kind, mb) that the device dispatcher (csrc/rrfp_exec.cu) selects with a
SWITCH node, so no host is involved per task.

Kernels: tcgen05/TMA GEMMs with fused bias / GELU / residual / GELU'
epilogues (csrc/gemm_sm100.cu), LayerNorm fwd/bwd, embedding and softmax
cross-entropy (csrc/ops.cu).  The attention core is the cuDNN SDPA kernel
(library, SURVEY.md K9 "library first").

The last kernel of a forward task writes its activation straight into the
next stage's mailbox slot (peer memory when stages live on different GPUs);
the last kernel of a backward task does the same with the input gradient.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K


@dataclass(frozen=True)
class GPTConfig:
    n_layer: int = 24
    d_model: int = 2048
    n_head: int = 16
    d_ff: int = 8192
    vocab: int = 50304
    seq: int = 2048
    eps: float = 1e-5
    init_std: float = 0.02
    causal: bool = True          # False: bidirectional attention (the ViT encoder of config 4)

    @property
    def d_head(self):
        return self.d_model // self.n_head

    def flops_per_layer(self, rows: int | None = None):
        """(F, B-input, W) matmul FLOPs of one layer for one microbatch of `rows` tokens."""
        s, d, f = rows or self.seq, self.d_model, self.d_ff
        gemm = 2 * s * d * (3 * d + d + 2 * f)
        attn = 2 * 2 * s * s * d / (2 if self.causal else 1)   # QK^T and PV (causal: half)
        return gemm + attn, gemm + 2 * attn, gemm

    def flops_head(self):
        return 2 * self.seq * self.d_model * self.vocab


GPT_1P3B = GPTConfig()
GPT_7B = GPTConfig(n_layer=32, d_model=4096, n_head=32, d_ff=16384)
VIT_H14 = GPTConfig(n_layer=32, d_model=1280, n_head=16, d_ff=5120, vocab=0, seq=2048, causal=False)


@dataclass(frozen=True)
class MultimodalSpec:
    """BASELINE config 4: a ViT encoder on the leading ``vit_stages`` pipeline
    stages feeding a GPT LLM.  Microbatch mb carries n_img(mb) ~ U{1..max_images}
    images (seeded, rng.substream(image_seed, "images", mb)), i.e. T_v(mb) =
    patch_tokens * n_img(mb) visual tokens: the ViT stages' work and their
    messages are input-dependent.  The LLM sequence is [projected visual
    tokens (T_v rows), text tokens (seq - T_v rows)]; loss over all positions.
    Patches are synthetic bf16 features [T_v, d_patch] (no pixels / network)."""
    vit: GPTConfig = VIT_H14
    llm: GPTConfig = GPT_7B
    vit_stages: int = 1
    patch_tokens: int = 256
    d_patch: int = 768
    max_images: int = 8
    image_seed: int = 0

    def images(self, n_mb: int):
        from .rng import substream
        return [int(substream(self.image_seed, "images", mb).integers(1, self.max_images + 1))
                for mb in range(n_mb)]

    def visual_tokens(self, n_mb: int):
        out = [self.patch_tokens * n for n in self.images(n_mb)]
        if max(out) > self.llm.seq or self.patch_tokens * self.max_images > self.vit.seq:
            raise ValueError("visual tokens exceed the sequence length")
        return out


def init_mm_params(spec: MultimodalSpec, device, seed: int, which: str):
    """Patch embedding ('pe': [d_vit, d_patch]) or projector ('proj': [d_llm, d_vit])."""
    g = _gen(device, seed * 100003 + (55551 if which == "pe" else 55553))
    bf = torch.bfloat16
    dv, dl = spec.vit.d_model, spec.llm.d_model
    if which == "pe":
        return {"w_pe": (torch.randn(dv, spec.d_patch, generator=g, device=device) * 0.02).to(bf),
                "b_pe": (torch.randn(dv, generator=g, device=device) * 0.02).to(bf)}
    return {"w_proj": (torch.randn(dl, dv, generator=g, device=device) * 0.02).to(bf),
            "b_proj": (torch.randn(dl, generator=g, device=device) * 0.02).to(bf)}


def synthetic_patches(spec: MultimodalSpec, n_mb: int, seed: int, device):
    g = _gen(device, seed * 7919 + 3)
    return (torch.randn(n_mb, spec.vit.seq, spec.d_patch, generator=g, device=device)).to(torch.bfloat16)


def split_layers(n_layer: int, n_stages: int, stage: int, head_cost: float = 0.0):
    """Global layer ids of `stage`.  head_cost = 0: even split (earlier stages
    take the remainder).  head_cost > 0: the last stage also runs the LM head +
    loss, worth `head_cost` layers; the split minimises the largest stage cost
    (the pipeline's bottleneck), e.g. 24 layers / 8 stages / head 1.5 ->
    [4,3,3,3,3,3,3,2] (max 4.0 layer-equivalents instead of 4.5)."""
    if head_cost <= 0 or n_stages == 1:
        counts = [n_layer // n_stages + (1 if s < n_layer % n_stages else 0) for s in range(n_stages)]
    else:
        m = max(1, math.ceil((n_layer + head_cost) / n_stages))
        while (n_stages - 1) * m + max(1, math.floor(m - head_cost)) < n_layer:
            m += 1
        last = max(1, min(math.floor(m - head_cost), n_layer - (n_stages - 1)))
        rest = n_layer - last
        counts = [rest // (n_stages - 1) + (1 if s < rest % (n_stages - 1) else 0)
                  for s in range(n_stages - 1)] + [last]
    lo = sum(counts[:stage])
    return list(range(lo, lo + counts[stage]))


ATTN_KEYS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o")
MLP_KEYS = ("ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")
# attention half's share of a layer's F+B time (LN1 + QKV + SDPA + out-proj vs LN2 +
# FC1 + FC2): 8·S·D² + 2·S²·D of 26·S·D² matmul FLOPs at S = D (0.385), raised for the
# SDPA kernels' lower efficiency than the GEMMs' -- measured F+B per half-layer on 16
# SMs (profiles/r01_emulated_pp8_half.json)
ATTN_FRAC = 0.42


def split_units(n_layer: int, n_stages: int, stage: int, head_cost: float = 0.0,
                split: str = "layer", attn_frac: float = ATTN_FRAC):
    """This stage's share of the model as [(global layer, part)], part "full" /
    "attn" (LN1 -> QKV -> attention -> out-proj + residual) / "mlp" (LN2 -> FC1
    -> GELU -> FC2 + residual).

    split "layer": whole layers, split_layers().  split "half": stage boundaries
    may also fall between a layer's attention and MLP halves (the residual
    stream crossing there is the same [S, D] activation the mailbox carries at a
    layer boundary); the contiguous partition of the 2·L half-layer units (+ the
    LM head on the last stage) minimises the largest stage cost, then the sum of
    squared stage costs.  24 layers / 8 stages / head 1.4: bottleneck 3.32
    layer-equivalents instead of 4.0."""
    if split == "layer":
        return [(l, "full") for l in split_layers(n_layer, n_stages, stage, head_cost)]
    if split != "half":
        raise ValueError("split must be 'layer' or 'half'")
    units = [(l, part) for l in range(n_layer) for part in ("attn", "mlp")]
    cost = [attn_frac if part == "attn" else 1.0 - attn_frac for _, part in units]
    bounds = _balanced_partition(cost, n_stages, head_cost, os.environ.get("RRFP_SPLIT_ORDER", "front") == "front")
    own = units[bounds[stage]:bounds[stage + 1]]
    out = []
    for l, part in own:            # attn + mlp of one layer on one stage = "full"
        if out and out[-1][0] == l:
            out[-1] = (l, "full")
        else:
            out.append((l, part))
    return out


def _balanced_partition(cost, n, tail, front: bool = True):
    """Cut points b[0..n] of `cost` into n non-empty contiguous segments (the last
    one also carries `tail`): min over partitions of the max segment cost, ties
    broken by the smallest sum of squares, then (front) by putting the heavier
    segments first -- a pipeline's first stages never wait for an activation,
    so excess work costs least there.  O(n·U²), U = len(cost)."""
    U = len(cost)
    if U < n:
        raise ValueError(f"{U} units cannot fill {n} stages")
    pre = [0.0]
    for c in cost:
        pre.append(pre[-1] + c)
    seg = lambda i, j, k: pre[j] - pre[i] + (tail if k == n - 1 else 0.0)
    INF = float("inf")

    def solve(key, cap):
        # best[k][j]: the first j units in k+1 segments; key(acc, segment cost, k)
        best = [[INF] * (U + 1) for _ in range(n)]
        arg = [[-1] * (U + 1) for _ in range(n)]
        for j in range(1, U + 1):
            c = seg(0, j, 0)
            if c <= cap:
                best[0][j], arg[0][j] = key(0.0, c, 0), 0
        for k in range(1, n):
            for j in range(k + 1, U + 1):
                for i in range(k, j):
                    c = seg(i, j, k)
                    if best[k - 1][i] == INF or c > cap:
                        continue
                    v = key(best[k - 1][i], c, k)
                    if v < best[k][j] - 1e-12:
                        best[k][j], arg[k][j] = v, i
        b, j = [U], U
        for k in range(n - 1, 0, -1):
            j = arg[k][j]
            b.append(j)
        return best[n - 1][U], [0] + b[::-1]

    m, _ = solve(lambda acc, c, k: max(acc, c), INF)
    bias = 1e-4 if front else 0.0
    _, bounds = solve(lambda acc, c, k: acc + c * c + bias * k * c, m + 1e-9)
    return bounds


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def init_layer_params(cfg: GPTConfig, layer: int, device, seed: int):
    """Deterministic per GLOBAL layer index, so every PP split sees the same model."""
    g = _gen(device, seed * 100003 + layer)
    d, f = cfg.d_model, cfg.d_ff
    std, out_std = cfg.init_std, cfg.init_std / math.sqrt(2 * cfg.n_layer)
    bf = torch.bfloat16

    def n(*shape, s=std):
        return (torch.randn(*shape, generator=g, device=device) * s).to(bf)

    def small(*shape):
        return (torch.randn(*shape, generator=g, device=device) * 0.02).to(bf)

    return {
        "ln1_g": (1.0 + small(d).float()).to(bf), "ln1_b": small(d),
        "w_qkv": n(3 * d, d), "b_qkv": small(3 * d),
        "w_o": n(d, d, s=out_std), "b_o": small(d),
        "ln2_g": (1.0 + small(d).float()).to(bf), "ln2_b": small(d),
        "w_1": n(f, d), "b_1": small(f),
        "w_2": n(d, f, s=out_std), "b_2": small(d),
    }


def shard_layer_params(cfg: GPTConfig, p: dict, rank: int, size: int) -> dict:
    """Megatron split of one layer over a TP group of `size` ranks: QKV and FC1
    column-parallel (heads / FFN columns rank*1/size..), out-proj and FC2
    row-parallel (their input features); LayerNorms and the row-parallel biases
    b_o, b_2 replicated (added once, inside the all-reduce)."""
    if size == 1:
        return p
    D, Fd = cfg.d_model, cfg.d_ff
    dl, fl = D // size, Fd // size
    q = slice(rank * dl, (rank + 1) * dl)
    f = slice(rank * fl, (rank + 1) * fl)
    out = dict(p)
    out["w_qkv"] = torch.cat([p["w_qkv"][i * D:(i + 1) * D][q] for i in range(3)]).contiguous()
    out["b_qkv"] = torch.cat([p["b_qkv"][i * D:(i + 1) * D][q] for i in range(3)]).contiguous()
    out["w_o"] = p["w_o"][:, q].contiguous()
    out["w_1"] = p["w_1"][f].contiguous()
    out["b_1"] = p["b_1"][f].contiguous()
    out["w_2"] = p["w_2"][:, f].contiguous()
    return out


def init_embed_params(cfg: GPTConfig, device, seed: int):
    g = _gen(device, seed * 100003 + 77777)
    bf = torch.bfloat16
    return {"wte": (torch.randn(cfg.vocab, cfg.d_model, generator=g, device=device) * cfg.init_std).to(bf),
            "wpe": (torch.randn(cfg.seq, cfg.d_model, generator=g, device=device) * cfg.init_std).to(bf)}


def init_head_params(cfg: GPTConfig, device, seed: int):
    g = _gen(device, seed * 100003 + 99991)
    bf = torch.bfloat16
    d = cfg.d_model
    return {"lnf_g": (1.0 + 0.02 * torch.randn(d, generator=g, device=device)).to(bf),
            "lnf_b": (0.02 * torch.randn(d, generator=g, device=device)).to(bf),
            "w_lm": (torch.randn(cfg.vocab, d, generator=g, device=device) * cfg.init_std).to(bf)}


def synthetic_batch(cfg: GPTConfig, n_mb: int, seed: int, device):
    """Tokens / next-token targets uniform in [0, V) from torch.Generator(seed)."""
    g = _gen(device, seed)
    toks = torch.randint(0, cfg.vocab, (n_mb, cfg.seq + 1), generator=g, device=device,
                         dtype=torch.int32)
    return toks[:, :-1].contiguous(), toks[:, 1:].contiguous()


def _ln_fwd(x, g, b, y, mean, rstd, eps):
    K.note()
    L = _lib.lib()
    _lib.check(L.rrfp_layernorm_fwd(K._p(x), K._p(g), K._p(b), K._p(y), K._p(mean), K._p(rstd),
                                    x.shape[0], x.shape[1], C.c_float(eps), K._stream()))


def _ln_bwd(dy, x, mean, rstd, g, dres, dx, dg, db):
    K.note((dx is not None) + (dg is not None or db is not None))   # dx kernel + parameter kernel
    L = _lib.lib()
    _lib.check(L.rrfp_layernorm_bwd(K._p(dy), K._p(x), K._p(mean), K._p(rstd), K._p(g),
                                    K._p(dres), K._p(dx), K._p(dg), K._p(db), x.shape[0],
                                    x.shape[1], K._stream()))


def _ln_bwd_fused(dy, x, mean, rstd, g, dres, dx, dg=None, db=None, cs_res=None, cs_dx=None):
    """One-pass LayerNorm backward (csrc/ops.cu ln_bwd_fused_kernel): dx (+ dres),
    the LN parameter gradients and the column sums of dres / dx (the bias
    gradients of the adjacent linear layers) in one kernel."""
    K.note()
    _lib.check(_lib.lib().rrfp_layernorm_bwd_fused(
        K._p(dy), K._p(x), K._p(mean), K._p(rstd), K._p(g), K._p(dres), K._p(dx), K._p(dg), K._p(db),
        K._p(cs_res), K._p(cs_dx), dy.shape[0], dy.shape[1], K._stream()))


def _copy_rows(dst, src, rows, cols):
    """bf16 [rows, cols] copy (e.g. into a peer stage's mailbox slot)."""
    K.note()
    _lib.check(_lib.lib().rrfp_copy_rows(
        C.c_void_p(dst.data_ptr()), C.c_longlong(dst.stride(0) * 2), C.c_void_p(src.data_ptr()),
        C.c_longlong(src.stride(0) * 2), rows, C.c_longlong(cols * 2), K._stream()))


def _bias_grad(dy, db):
    K.note()
    _lib.check(_lib.lib().rrfp_bias_grad(K._p(dy), C.c_longlong(dy.stride(0)), K._p(db),
                                         dy.shape[0], dy.shape[1], K._stream()))


class RawBuffer:
    """A device buffer given by address (e.g. a peer mailbox opened over CUDA IPC)."""

    def __init__(self, ptr: int, shape, stride0):
        self.ptr, self.shape, self._s0 = ptr, tuple(shape), stride0

    def data_ptr(self):
        return self.ptr

    def stride(self, i):
        return self._s0 if i == 0 else 1


def _half(p: dict, part: str) -> dict:
    """The parameters a (half-)layer holds on this stage."""
    if part == "full":
        return p
    return {k: p[k] for k in (ATTN_KEYS if part == "attn" else MLP_KEYS)}


class StageCompute:
    def __init__(self, cfg: GPTConfig, stage: int, n_stages: int, n_mb: int, device, *,
                 decompose: bool = False, seed: int = 1234, data_seed: int = 0,
                 fwd_in=None, bwd_in=None, tp_rank: int = 0, tp_size: int = 1, tp=None,
                 mm: MultimodalSpec | None = None, head_cost: float = 0.0, w_split: str = "fc",
                 split: str = "layer", attn_frac: float = ATTN_FRAC):
        self.cfg, self.stage, self.n_stages, self.M = cfg, stage, n_stages, n_mb
        self.device = torch.device(device)
        self.decompose = decompose
        if w_split not in ("fc", "all"):
            raise ValueError("w_split must be 'fc' or 'all'")
        # decomposed backward: which weight gradients the W task takes -- "fc": FC1/FC2
        # (default; the attention ones overlap the attention backward in B), "all": all four
        self.w_split = w_split
        self.mm = mm
        # which part of the model this stage holds (config 4: ViT stages, then LLM stages)
        if mm is not None:
            nv = mm.vit_stages
            part, idx, cnt = ("vit", stage, nv) if stage < nv else ("llm", stage - nv, n_stages - nv)
            if cfg != (mm.vit if part == "vit" else mm.llm):
                raise ValueError(f"stage {stage} ({part}) needs cfg = mm.{part}")
            if tp_size > 1:
                raise ValueError("the multimodal path has no TP split")
        else:
            part, idx, cnt = "gpt", stage, n_stages
        self.part = part
        # head_cost > 0: balance the layer split against the last stage's LM head;
        # split "half": stage boundaries may fall inside a layer (split_units), so
        # the first layer may be its MLP half only and the last its attention half
        if split != "layer" and part != "gpt":
            raise ValueError("split='half' is for the GPT pipeline (not config 4)")
        units = split_units(cfg.n_layer, cnt, idx, head_cost if part != "vit" else 0.0, split, attn_frac)
        self.layers = [l for l, _ in units]
        self.parts = [pt for _, pt in units]
        # prologue: token embedding (GPT stage 0), patch embedding (ViT stage 0), or
        # merge (first LLM stage: projected visual rows arrive in the mailbox, text
        # rows are embedded here); epilogue: LM head + loss, or the ViT projector
        self.prologue = {"gpt": "tokens", "vit": "patches", "llm": "merge"}[part] if idx == 0 else None
        self.epilogue = ("projector" if part == "vit" else "head") if idx == cnt - 1 else None
        self.first = self.prologue in ("tokens", "patches")
        self.last = self.epilogue == "head"
        S, D, Fd, V = cfg.seq, cfg.d_model, cfg.d_ff, cfg.vocab
        self.T_v = mm.visual_tokens(n_mb) if mm is not None else None
        # rows each microbatch occupies in this stage's layers (ViT: its visual tokens)
        self.rows = list(self.T_v) if part == "vit" else [S] * n_mb
        if cfg.n_head % tp_size or Fd % tp_size:
            raise ValueError(f"TP size {tp_size} must divide n_head and d_ff")
        if tp_size > 1 and tp is None:
            raise ValueError("tp_size > 1 needs a TpComm (paper_2605_18750_b200.tp)")
        # tensor parallelism (config 3): this rank's heads / FFN columns
        self.tp_rank, self.R, self.tp = tp_rank, tp_size, tp
        self.model_seed = seed
        self.Hl, self.Dl, self.Fl = cfg.n_head // tp_size, D // tp_size, Fd // tp_size
        Dl, Fl = self.Dl, self.Fl
        dev, bf = self.device, torch.bfloat16
        lseed = seed + 17 if part == "vit" else seed      # ViT layers: their own init stream
        self.layer_seed = lseed
        with torch.no_grad():
            self.p = [_half(shard_layer_params(cfg, init_layer_params(cfg, l, dev, lseed), tp_rank, tp_size), pt)
                      for l, pt in units]
            self.emb = init_embed_params(cfg, dev, seed) if self.prologue in ("tokens", "merge") else None
            self.head = init_head_params(cfg, dev, seed) if self.last else None
            self.pe = init_mm_params(mm, dev, seed, "pe") if self.prologue == "patches" else None
            self.proj = init_mm_params(mm, dev, seed, "proj") if self.epilogue == "projector" else None
        # every fp32 gradient is a view of ONE flat buffer (each view 1 KiB aligned for
        # the TMA reduce-add epilogues), so zero_grads() is a single memset
        groups = [*self.p, self.emb, self.head, self.pe, self.proj]
        align = 256
        total = sum((v.numel() + align - 1) // align * align for d in groups if d for v in d.values())
        self.grad_flat = torch.zeros(max(total, 1), device=dev)
        off = [0]

        def zeros(d):
            if not d:
                return None
            out = {}
            for k, v in d.items():
                out[k] = self.grad_flat[off[0]:off[0] + v.numel()].view(v.shape)
                off[0] += (v.numel() + align - 1) // align * align
            return out
        self.g = [zeros(p) for p in self.p]
        self.g_emb, self.g_head = zeros(self.emb), zeros(self.head)
        self.g_pe, self.g_proj = zeros(self.pe), zeros(self.proj)
        # synthetic data (tokens where the sequence starts, targets at the loss, patches for the ViT)
        if part != "vit":
            toks, tgts = synthetic_batch(cfg, n_mb, data_seed, dev)
            self.tokens = toks if self.prologue in ("tokens", "merge") else None
            self.targets = tgts if self.last else None
        else:
            self.tokens = self.targets = None
        self.patches = synthetic_patches(mm, n_mb, data_seed, dev) if self.prologue == "patches" else None
        # mailboxes written by neighbours: F input (stage > 0), B input (stage < N-1)
        # (the caller may pass IPC-exportable buffers, distributed.py); the ViT
        # projector stage receives the gradient of its [T_v, d_llm] output
        if fwd_in is None and not self.first:
            fwd_in = torch.empty(n_mb, S, D, device=dev, dtype=bf)
        if bwd_in is None and not self.last:
            bw = mm.llm.d_model if self.epilogue == "projector" else D
            bwd_in = torch.empty(n_mb, S, bw, device=dev, dtype=bf)
        self.fwd_in, self.bwd_in = fwd_in, bwd_in
        self.fwd_out = None   # per-mb destination buffers (set by connect_outputs)
        self.bwd_out = None
        # activation slots, one per microbatch (static addresses for graph capture)
        nl = len(self.layers)
        e = lambda *s: torch.empty(*s, device=dev, dtype=bf)
        f32 = lambda *s: torch.empty(*s, device=dev, dtype=torch.float32)
        self.x0 = e(n_mb, S, D) if self.first else None
        self.h1, self.qkv, self.x2 = e(n_mb, nl, S, D), e(n_mb, nl, S, 3 * Dl), e(n_mb, nl, S, D)
        # (the attention output lives in cuDNN's BSHD output buffer, see _attn_fwd)
        self.h2, self.pre, self.act, self.y = e(n_mb, nl, S, D), e(n_mb, nl, S, Fl), e(n_mb, nl, S, Fl), e(n_mb, nl, S, D)
        self.m1, self.r1, self.m2, self.r2 = f32(n_mb, nl, S), f32(n_mb, nl, S), f32(n_mb, nl, S), f32(n_mb, nl, S)
        self.attn_aux = [[None] * nl for _ in range(n_mb)]
        self.o_view = [[None] * nl for _ in range(n_mb)]   # attention output as [S, D]
        # attention core: cuDNN SDPA through the frontend graph API (attention.py) reading
        # the packed QKV and writing O / stats / packed dQKV into our own slots;
        # RRFP_ATTN=torch selects the aten op (separate dQ/dK/dV, copied in)
        # RRFP_LN_FUSED=1: LayerNorm parameter gradients fused with the adjacent bias
        # gradients (column sums of the residual gradients) in one side-stream pass
        # (ops.cu ln_bwd_fused_kernel), the head's LN backward in one kernel.
        # Off by default: alone the fused pass takes 8.8 us against 15.6 for the two kernels
        # it replaces (tools/ln_bench.py), but inside the task bodies the separate, smaller
        # kernels fill the weight-gradient GEMMs' tails better: W 118.5 vs 124.5 us/layer,
        # fused B 390.7 vs 394.2 (tools/task_times.py 9 [bfw], same box, interleaved)
        self.ln_fused = os.environ.get("RRFP_LN_FUSED", "0") == "1" and D <= 4096
        # FC1 bias gradient reduced in the FC2-dgrad GEMM epilogue (EPI_GELU_BWD + C2):
        # off by default -- the main-chain GEMM's epilogue got ~2.6 us/layer slower, more
        # than the separate column-sum kernel costs on the side stream (B 12,207 vs
        # 12,144 us per microbatch at PP=1); RRFP_COLSUM_EPI=1 selects it
        self.colsum_epi = os.environ.get("RRFP_COLSUM_EPI", "0") == "1"
        self.attn_impl = os.environ.get("RRFP_ATTN", "cudnn_fe")
        self._sdpa = {}
        if self.attn_impl == "cudnn_fe" and nl:
            from .attention import sdpa_graphs
            self.attn_o = e(n_mb, nl, S, Dl)
            self.attn_st = f32(n_mb, nl, self.Hl, S)
            for T in sorted(set(self.rows)):
                self._sdpa[T] = sdpa_graphs(T, self.Hl, cfg.d_head, cfg.causal, dev, S)
            ws = max(g.workspace_bytes for g in self._sdpa.values())
            self.attn_ws = torch.empty(max(ws, 16), device=dev, dtype=torch.uint8)
        # forward attention core: our tcgen05 kernel (csrc/fmha_sm100.cu) for d_head 128
        # (GPT-1.3B / 7B); its softmax statistics are the layout cuDNN's backward reads
        self.own_attn_fwd = (bool(self._sdpa) and cfg.d_head == 128 and all(T % 128 == 0 for T in self.rows)
                             and os.environ.get("RRFP_ATTN_FWD", "own") == "own")
        # backward: our kernel on RRFP_ATTN_BWD=own (parity-tested; on the 1.3B shape it
        # measures 82 us against cuDNN's 66 us, so cuDNN's backward is the default)
        self.own_attn_bwd = self.own_attn_fwd and os.environ.get("RRFP_ATTN_BWD", "cudnn") == "own"
        if self.own_attn_bwd:
            self.attn_bwd_ws = K.attn_bwd_workspace(S, self.Hl, dev)
        if self.last:
            self.hf, self.mf, self.rf = e(n_mb, S, D), f32(n_mb, S), f32(n_mb, S)
            self.logits = e(n_mb, S, V)
            self.loss = torch.zeros(n_mb, S, device=dev)
            self.lse = f32(n_mb, S)
            # LM head + cross-entropy forward fused (gemm EPI_BF16_LSE + xent_combine);
            # RRFP_CE_FUSED=0: GEMM, then xent_fwd over the logits
            self.ce_fused = os.environ.get("RRFP_CE_FUSED", "1") != "0" and V % 8 == 0
            self.ce_part = f32(S, K.lm_head_slots(V), 2) if self.ce_fused else None   # shared scratch
        # scratch shared by all bodies of this stage (bodies never overlap on a lane)
        # two parity sets (layer li uses set li % 2) so the weight-gradient
        # GEMMs of layer li can run on the side stream while layer li-1's
        # input-gradient chain proceeds on the main stream
        self.sd_a = [e(S, D), e(S, D)]
        self.sd_b = [e(S, D), e(S, D)]
        self.sd_big = [e(S, Fl), e(S, Fl)]
        self.sd_qkv = [e(S, 3 * Dl), e(S, 3 * Dl)]
        # LayerNorm input gradients, kept (two parity sets) until the side stream's
        # parameter-gradient kernels read them (fused backward; decomposed: gln1/gln2)
        if not decompose:
            self.sd_ln1, self.sd_ln2 = [e(S, D), e(S, D)], [e(S, D), e(S, D)]
        self.d_head = e(S, D)
        self.d_o = e(S, Dl) if tp_size > 1 else None   # attention-output gradient (this rank's heads)
        self.side = torch.cuda.Stream(dev)
        if decompose:   # gradients kept per (mb, layer) for the deferred W task
            self.gy, self.gpre = e(n_mb, nl, S, D), e(n_mb, nl, S, Fl)
            # LayerNorm input gradients (the LN1 / LN2 parameter gradients move to W)
            self.gln1, self.gln2 = e(n_mb, nl, S, D), e(n_mb, nl, S, D)
            self.gx0 = e(n_mb, S, D) if self.prologue else None
            if w_split == "all":
                self.gx2, self.gqkv = e(n_mb, nl, S, D), e(n_mb, nl, S, 3 * Dl)
        self.graphs = {}
        self.kernel_counts = {}   # (kind, mb) -> our kernel launches in that body
        self.gemm_sm_cap = 0      # > 0: GEMM grids confined to this many SMs (see run_task)

    # ------------------------------------------------------------ wiring
    def connect_outputs(self, fwd_out=None, bwd_out=None):
        """fwd_out / bwd_out: per-mb destination (tensor or RawBuffer) in the
        next / previous stage's mailbox, or per-mb LISTS of destinations (one per
        TP rank of the neighbour stage; a TP rank keeps only its own rank's)."""
        as_list = lambda v: v if isinstance(v, (list, tuple)) else [v]

        def own_rank(lst):
            # the R ranks of a TP group hold bit-identical activations / input gradients
            # after the all-reduce (partials summed in rank order), so rank r feeds only
            # the neighbour's rank r (whose flag it raises anyway): half the NVLink
            # bytes of writing every receiver rank at TP=2 (RRFP_TP_ALL_RECEIVERS=1: all)
            if self.R > 1 and len(lst) == self.R and os.environ.get("RRFP_TP_ALL_RECEIVERS", "0") != "1":
                return [lst[self.tp_rank]]
            return lst
        self.fwd_out = [own_rank(as_list(v)) for v in fwd_out] if fwd_out is not None else None
        self.bwd_out = [own_rank(as_list(v)) for v in bwd_out] if bwd_out is not None else None

    def param_bytes(self):
        return sum(t.numel() * 2 for p in self.p for t in p.values())

    # ------------------------------------------------------------ forward
    def _attn_fwd(self, qkv, mb, li):
        T, H, Dh, D = qkv.shape[0], self.Hl, self.cfg.d_head, self.Dl
        if self.own_attn_fwd:
            o = self.attn_o[mb, li, :T]
            K.attn_fwd(qkv, o, self.attn_st[mb, li], heads=H, causal=self.cfg.causal, T=T)
            self.o_view[mb][li] = o
            return
        if self._sdpa:
            o = self.attn_o[mb, li, :T]
            self._sdpa[T].forward(qkv.data_ptr(), o.data_ptr(), self.attn_st[mb, li].data_ptr(),
                                  self.attn_ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
            self.o_view[mb][li] = o
            return
        q = qkv[:, :D].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        k = qkv[:, D:2 * D].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        v = qkv[:, 2 * D:].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        out = torch.ops.aten._scaled_dot_product_cudnn_attention(
            q, k, v, None, True, 0.0, self.cfg.causal, False, scale=1.0 / math.sqrt(Dh))
        o4, lse = out[0], out[1]
        self.attn_aux[mb][li] = (o4, lse, out[2], out[3], out[4], out[5], out[6], out[7])
        o_sd = o4[0].transpose(0, 1)
        if o_sd.is_contiguous():          # cuDNN writes BSHD: use it in place as [T, D]
            self.o_view[mb][li] = o_sd.reshape(T, D)
        else:
            o = torch.empty(T, D, device=self.device, dtype=torch.bfloat16)
            o.view(T, H, Dh).copy_(o_sd)
            self.o_view[mb][li] = o

    def _text_rows(self, mb):
        """First text row of microbatch mb in the LLM sequence (after its visual tokens)."""
        return self.T_v[mb] if self.prologue == "merge" else 0

    def forward(self, mb: int):
        cfg = self.cfg
        S, D = cfg.seq, cfg.d_model
        T = self.rows[mb]
        if self.prologue == "tokens":
            K.note()
            _lib.check(_lib.lib().rrfp_embedding_fwd(
                K._p(self.tokens[mb]), K._p(self.emb["wte"]), K._p(self.emb["wpe"]),
                K._p(self.x0[mb]), S, D, K._stream()))
            x = self.x0[mb]
        elif self.prologue == "patches":   # ViT patch embedding of this microbatch's images
            x = self.x0[mb, :T]
            K.gemm(self.patches[mb, :T], self.pe["w_pe"], x, bias=self.pe["b_pe"])
        else:
            x = self.fwd_in[mb][:T]
            t0 = self._text_rows(mb)
            if self.prologue == "merge" and t0 < S:   # text rows after the projected visual rows
                K.note()
                _lib.check(_lib.lib().rrfp_embedding_fwd(
                    K._p(self.tokens[mb, t0:]), K._p(self.emb["wte"]), K._p(self.emb["wpe"][t0:]),
                    K._p(x[t0:]), S - t0, D, K._stream()))
        for li, p in enumerate(self.p):
            part = self.parts[li]
            h1, qkv = self.h1[mb, li, :T], self.qkv[mb, li, :T]
            h2, pre, act = self.h2[mb, li, :T], self.pre[mb, li, :T], self.act[mb, li, :T]
            if part == "mlp":         # the attention half ran on the previous stage
                x2 = x
            else:
                # an attention half ending the stage writes the next stage's mailbox
                x2s = ([o[:T] for o in self._layer_output(mb, li)] if part == "attn"
                       else [self.x2[mb, li, :T]])
                x2 = x2s[0]
                _ln_fwd(x, p["ln1_g"], p["ln1_b"], h1, self.m1[mb, li, :T], self.r1[mb, li, :T], cfg.eps)
                K.gemm(h1, p["w_qkv"], qkv, bias=p["b_qkv"])
                self._attn_fwd(qkv, mb, li)
                if self.R == 1:
                    K.gemm(self.o_view[mb][li], p["w_o"], x2, epi=K.EPI_RESID, bias=p["b_o"], r=x,
                           m=T, n=D, k=self.Dl)
                else:   # row-parallel: partial sum, then all-reduce (+ b_o + residual) over the TP group
                    K.gemm(self.o_view[mb][li], p["w_o"], self.tp.partial, m=S, n=D, k=self.Dl)
                    self.tp.allreduce(x2s, bias=p["b_o"], resid=x)
                if part == "attn":
                    x = x2
                    continue
            _ln_fwd(x2, p["ln2_g"], p["ln2_b"], h2, self.m2[mb, li, :T], self.r2[mb, li, :T], cfg.eps)
            K.gemm(h2, p["w_1"], pre, epi=K.EPI_BIAS_GELU, c2=act, bias=p["b_1"])
            outs = [o[:T] for o in self._layer_output(mb, li)]   # last layer: next stage's mailbox
            if self.R == 1:
                K.gemm(act, p["w_2"], outs[0], epi=K.EPI_RESID, bias=p["b_2"], r=x2, m=T, n=D, k=self.Fl)
            else:
                K.gemm(act, p["w_2"], self.tp.partial, m=S, n=D, k=self.Fl)
                self.tp.allreduce(outs, bias=p["b_2"], resid=x2)
            x = outs[0]
        if self.last:
            h = self.head
            _ln_fwd(x, h["lnf_g"], h["lnf_b"], self.hf[mb], self.mf[mb], self.rf[mb], cfg.eps)
            if self.ce_fused:   # softmax statistics from the GEMM epilogue (no pass over the logits)
                K.lm_head_xent_fwd(self.hf[mb], h["w_lm"], self.logits[mb], self.targets[mb], self.loss[mb],
                                   self.lse[mb], self.ce_part)
            else:
                K.gemm(self.hf[mb], h["w_lm"], self.logits[mb])
                K.note()
                _lib.check(_lib.lib().rrfp_xent_fwd(
                    K._p(self.logits[mb]), C.c_longlong(cfg.vocab), K._p(self.targets[mb]), S,
                    cfg.vocab, K._p(self.loss[mb]), K._p(self.lse[mb]), K._stream()))
        elif self.epilogue == "projector":   # [T_v, d_vit] -> [T_v, d_llm] rows of the LLM mailbox
            for dst in self.fwd_out[mb]:
                K.gemm(x, self.proj["w_proj"], dst[:T], bias=self.proj["b_proj"])

    def _layer_input(self, mb, li):
        T = self.rows[mb]
        if li > 0:
            return self.y[mb, li - 1, :T]
        return self.x0[mb, :T] if self.first else self.fwd_in[mb][:T]

    def _layer_output(self, mb, li):
        """Destination list of layer li's output (the next stage's mailbox slot of
        every receiving TP rank for the last layer; first entry is read back)."""
        if (li == len(self.layers) - 1 and not self.last and self.epilogue != "projector"
                and self.fwd_out is not None):
            outs = list(self.fwd_out[mb])
            if len(outs) > 1 and self.R == 1:
                raise ValueError("a TP=1 stage feeds a TP>1 stage: not supported")
            return outs
        return [self.y[mb, li]]

    # ----------------------------------------------------------- backward
    def backward_input(self, mb: int):
        """B task: input gradients plus weight gradients; decomposed (BFW), the
        FC1/FC2 weight gradients (the larger half of the weight-gradient FLOPs)
        are deferred to the W task.

        Two streams: the input-gradient chain (dgrad GEMMs, LayerNorm and
        attention backward) runs on the main stream; each layer's weight-gradient
        GEMMs + bias reductions run on a side stream as soon as their inputs
        exist, so they fill the tail waves of the dgrad GEMMs and overlap the
        non-GEMM attention / LayerNorm backward; the LayerNorm parameter
        gradients join them there (from parity-buffered LN input gradients), so
        the main stream carries only the input-gradient chain.  That overlap is why the
        attention-side weight gradients stay in B even when decomposed: moved
        to W they would run alone (B-input + W > fused B).  Scratch comes in two
        parity sets; the main stream only rewrites a set after the side stream
        finished reading it (events).
        """
        cfg = self.cfg
        S, D, Fd, V = cfg.seq, cfg.d_model, cfg.d_ff, cfg.vocab
        T = self.rows[mb]
        dec = self.decompose
        fused_w = not dec          # FC1/FC2 (and head / prologue) weight gradients in this task
        nl = len(self.layers)
        main = torch.cuda.current_stream()
        side = self.side or main          # side=None: the whole task on one stream
        side_done = {}

        def ev():
            e = torch.cuda.Event()
            e.record(main)
            return e

        side_used = []

        def on_side(after, fn):
            if side == main:
                fn()
                return
            side_used.append(True)
            with torch.cuda.stream(side):
                side.wait_event(after)
                fn()

        def dy_buf(li):           # where layer li reads its output gradient
            return (self.gy[mb, li] if dec else self.sd_a[li % 2])[:T]

        if self.last:
            h, gh = self.head, self.g_head
            scale = 1.0 / (S * self.M)
            K.note()
            _lib.check(_lib.lib().rrfp_xent_bwd(
                K._p(self.logits[mb]), C.c_longlong(V), K._p(self.targets[mb]), S, V,
                K._p(self.lse[mb]), C.c_float(scale), K._stream()))
            if fused_w:
                on_side(ev(), lambda: K.gemm(self.logits[mb], self.hf[mb], gh["w_lm"], epi=K.EPI_ACC_F32,
                                             a_mn=True, b_mn=True, accumulate=True, m=V, n=D, k=S))
            K.gemm(self.logits[mb], h["w_lm"], self.d_head, b_mn=True, m=S, n=D, k=V)
            dy = dy_buf(nl - 1)
            (_ln_bwd_fused if self.ln_fused else _ln_bwd)(
                self.d_head, self.y[mb, nl - 1], self.mf[mb], self.rf[mb], h["lnf_g"], None, dy,
                gh["lnf_g"], gh["lnf_b"])
        elif self.epilogue == "projector":
            # gradient of the projected visual rows -> ViT output gradient (+ projector grads)
            dyp, pj, gp = self.bwd_in[mb][:T], self.proj, self.g_proj
            if fused_w:
                yl = self.y[mb, nl - 1, :T]
                on_side(ev(), lambda: (K.gemm(dyp, yl, gp["w_proj"], epi=K.EPI_ACC_F32, a_mn=True,
                                              b_mn=True, accumulate=True, m=dyp.shape[1], n=D, k=T),
                                       _bias_grad(dyp, gp["b_proj"])))
            dy = dy_buf(nl - 1)
            K.gemm(dyp, pj["w_proj"], dy, b_mn=True, m=T, n=D, k=dyp.shape[1])
        else:
            dy = self.bwd_in[mb][:T]   # (the W task reads it there too: a slot per microbatch)
        Dl, Fl = self.Dl, self.Fl
        d_head = self.d_head[:T]
        def stage_dx():
            """Destination of the stage's input gradient (+ the other TP ranks' copies)."""
            if self.prologue is None:
                if self.bwd_out is not None:
                    return self.bwd_out[mb][0][:T], [o[:T] for o in self.bwd_out[mb][1:]]
                dx = self.sd_a[1][:T]
            else:   # prologue stages keep the input gradient for the embedding backward
                dx = (self.gx0[mb] if dec else self.sd_a[1])[:T]
            if 1 in side_done:   # layer 1's side work read sd_a[1]
                main.wait_event(side_done[1])
            return dx, []

        for li in reversed(range(nl)):
            p, g = self.p[li], self.g[li]
            part = self.parts[li]
            x = self._layer_input(mb, li)
            h1, h2 = self.h1[mb, li, :T], self.h2[mb, li, :T]
            x2 = x if part == "mlp" else self.x2[mb, li, :T]
            pre, act = self.pre[mb, li, :T], self.act[mb, li, :T]
            q = li % 2
            if li + 2 in side_done:          # set q was last read by layer li+2's side work
                main.wait_event(side_done[li + 2])
            d_pre = (self.gpre[mb, li] if dec else self.sd_big[q])[:T]
            defer_attn = dec and self.w_split == "all"
            d_x2 = (self.gx2[mb, li] if defer_attn else self.sd_b[q])[:T]
            d_qkv = (self.gqkv[mb, li] if defer_attn else self.sd_qkv[q])[:T]
            extra = []
            if part == "attn":   # the MLP half is on the next stage: dy is the gradient of x2
                if defer_attn:
                    d_x2.copy_(dy)
                else:
                    d_x2 = dy
            else:
                if part == "mlp":    # (always the stage's first layer) LN2 backward ends the stage
                    d_x2, extra = stage_dx()
                if fused_w:
                    dyy = dy
                    on_side(ev(), lambda: (K.gemm(dyy, act, g["w_2"], epi=K.EPI_ACC_F32,
                                                  a_mn=True, b_mn=True, accumulate=True, m=D, n=Fl, k=T),
                                           None if self.ln_fused else _bias_grad(dyy, g["b_2"])))   # (b_2: LN2 side pass)
                # FC2 dgrad fused with GELU': d_pre = (dy . W2) * gelu'(pre)   (this rank's FFN columns)
                # (+ b_1's gradient, the column sums of d_pre, reduced in the same epilogue)
                K.gemm(dy, p["w_2"], d_pre, epi=K.EPI_GELU_BWD, b_mn=True, r=pre, m=T, n=Fl, k=D,
                       c2=g["b_1"] if self.colsum_epi else None)
                if fused_w:
                    on_side(ev(), lambda: (K.gemm(d_pre, h2, g["w_1"], epi=K.EPI_ACC_F32,
                                                  a_mn=True, b_mn=True, accumulate=True, m=Fl, n=D, k=T),
                                           None if self.colsum_epi else _bias_grad(d_pre, g["b_1"])))
                # FC1 dgrad (a partial sum under TP: all-reduced) -> LN2 backward (+ residual grad dy).
                # The LN2 parameter gradients leave the input-gradient chain: side stream
                # (fused), W task (decomposed, from the saved gln2)
                ln_dy = (self.gln2[mb, li] if dec else self.sd_ln2[q])[:T]
                self._dgrad_reduce(d_pre, p["w_1"], Fl, T, out=ln_dy)
                _ln_bwd(ln_dy, x2, self.m2[mb, li, :T], self.r2[mb, li, :T], p["ln2_g"], dy, d_x2, None, None)
                if not dec and self.ln_fused:
                    # side pass: LN2 parameter gradients + b_2's gradient (column sum of dy), one kernel
                    on_side(ev(), lambda ln_dy=ln_dy, x2=x2, g=g, li=li, dyy=dy: _ln_bwd_fused(
                        ln_dy, x2, self.m2[mb, li, :T], self.r2[mb, li, :T], None, dyy, None,
                        g["ln2_g"], g["ln2_b"], g["b_2"]))
                elif not dec:
                    on_side(ev(), lambda ln_dy=ln_dy, x2=x2, g=g, li=li: _ln_bwd(
                        ln_dy, x2, self.m2[mb, li, :T], self.r2[mb, li, :T], None, None, None,
                        g["ln2_g"], g["ln2_b"]))
                if part == "mlp":
                    for dst in extra:   # the other TP ranks of the previous stage (identical bytes)
                        _copy_rows(dst, d_x2, T, D)
                    dy = d_x2
                    continue
            ov = self.o_view[mb][li]
            if not defer_attn:
                dxx = d_x2
                on_side(ev(), lambda: (K.gemm(dxx, ov, g["w_o"], epi=K.EPI_ACC_F32,
                                              a_mn=True, b_mn=True, accumulate=True, m=D, n=Dl, k=T),
                                       None if self.ln_fused and not dec else _bias_grad(dxx, g["b_o"])))
            # out-proj dgrad -> attention backward -> QKV dgrad
            d_o = d_head if self.R == 1 else self.d_o
            K.gemm(d_x2, p["w_o"], d_o, b_mn=True, m=T, n=Dl, k=D)
            self._attn_bwd(mb, li, d_o, d_qkv)
            def qkv_w(d_qkv=d_qkv, h1=h1, g=g):
                K.gemm(d_qkv, h1, g["w_qkv"], epi=K.EPI_ACC_F32, a_mn=True,
                       b_mn=True, accumulate=True, m=3 * Dl, n=D, k=T)
                _bias_grad(d_qkv, g["b_qkv"])
            if not defer_attn:
                on_side(ev(), qkv_w)
            ln_dy = (self.gln1[mb, li] if dec else self.sd_ln1[q])[:T]
            self._dgrad_reduce(d_qkv, p["w_qkv"], 3 * Dl, T, out=ln_dy)
            # LN1 backward (+ residual d_x2) -> gradient of the layer input
            if li > 0:
                dx = dy_buf(li - 1)
                if li + 1 in side_done:   # layer li+1's side work read this buffer
                    main.wait_event(side_done[li + 1])
            else:
                dx, extra = stage_dx()
            _ln_bwd(ln_dy, x, self.m1[mb, li, :T], self.r1[mb, li, :T], p["ln1_g"], d_x2, dx, None, None)
            if not dec and self.ln_fused:
                # side pass: LN1 parameter gradients + b_o's gradient (column sum of d_x2), one kernel
                on_side(ev(), lambda ln_dy=ln_dy, x=x, g=g, li=li, dxx=d_x2: _ln_bwd_fused(
                    ln_dy, x, self.m1[mb, li, :T], self.r1[mb, li, :T], None, dxx, None,
                    g["ln1_g"], g["ln1_b"], g["b_o"]))
            elif not dec:
                on_side(ev(), lambda ln_dy=ln_dy, x=x, g=g, li=li: _ln_bwd(
                    ln_dy, x, self.m1[mb, li, :T], self.r1[mb, li, :T], None, None, None,
                    g["ln1_g"], g["ln1_b"]))
            if not defer_attn:   # everything this layer queued on the side stream (scratch set q)
                done = torch.cuda.Event()
                done.record(side)
                side_done[li] = done
            for dst in extra:   # the other TP ranks of the previous stage (identical bytes)
                _copy_rows(dst, dx, T, D)
            dy = dx
        if self.prologue == "merge":   # visual rows' gradient -> the ViT projector stage
            t0 = self._text_rows(mb)
            if self.bwd_out is not None:
                for dst in self.bwd_out[mb]:
                    _copy_rows(dst[:t0], dy[:t0], t0, D)
        if self.prologue and fused_w:
            dyy = dy
            on_side(ev(), lambda: self._prologue_wgrad(mb, dyy))
        if side_used:   # (a side stream never forked into a capture must not be joined)
            join = torch.cuda.Event()
            join.record(side)
            main.wait_event(join)

    def _prologue_wgrad(self, mb, dx):
        """Parameter gradients of the stage prologue from the input gradient dx."""
        S, D = self.cfg.seq, self.cfg.d_model
        T = self.rows[mb]
        if self.prologue == "patches":
            K.gemm(dx, self.patches[mb, :T], self.g_pe["w_pe"], epi=K.EPI_ACC_F32, a_mn=True, b_mn=True,
                   accumulate=True, m=D, n=self.mm.d_patch, k=T)
            _bias_grad(dx, self.g_pe["b_pe"])
            return
        t0 = self._text_rows(mb)
        if t0 >= S:
            return
        K.note()
        _lib.check(_lib.lib().rrfp_embedding_bwd(
            K._p(self.tokens[mb, t0:]), K._p(dx[t0:]), K._p(self.g_emb["wte"]),
            K._p(self.g_emb["wpe"][t0:]), S - t0, D, K._stream()))

    def _dgrad_reduce(self, d_col, w, k, T=None, out=None):
        """Input gradient of a column-parallel layer into `out` (default self.d_head):
        d_col . W (K = this rank's columns); under TP a partial sum all-reduced over the group."""
        S, D = self.cfg.seq, self.cfg.d_model
        T = S if T is None else T
        out = self.d_head if out is None else out
        if self.R == 1:
            K.gemm(d_col, w, out[:T], b_mn=True, m=T, n=D, k=k)
        else:
            K.gemm(d_col, w, self.tp.partial, b_mn=True, m=S, n=D, k=k)
            self.tp.allreduce([out])

    def _attn_bwd(self, mb, li, d_o, d_qkv):
        cfg = self.cfg
        T, H, Dh, D = d_qkv.shape[0], self.Hl, cfg.d_head, self.Dl
        qkv = self.qkv[mb, li, :T]
        if self.own_attn_bwd:
            K.attn_bwd(qkv, self.o_view[mb][li], d_o, self.attn_st[mb, li], d_qkv, self.attn_bwd_ws, heads=H,
                       causal=cfg.causal, T=T)
            return
        if self._sdpa:   # dQ, dK, dV straight into the packed gradient the QKV GEMMs read
            self._sdpa[T].backward(qkv.data_ptr(), self.o_view[mb][li].data_ptr(), d_o.data_ptr(),
                                   self.attn_st[mb, li].data_ptr(), d_qkv.data_ptr(),
                                   self.attn_ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
            return
        q = qkv[:, :D].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        k = qkv[:, D:2 * D].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        v = qkv[:, 2 * D:].view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        o4, lse, cq, ck, mq, mk, ps, po = self.attn_aux[mb][li]
        go = d_o.view(T, H, Dh).transpose(0, 1).unsqueeze(0)
        dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
            go, q, k, v, o4, lse, ps, po, None, cq, ck, mq, mk, 0.0,
            cfg.causal, scale=1.0 / math.sqrt(Dh))
        for i, t in enumerate((dq, dk, dv)):
            t_sd = t[0].transpose(0, 1)
            if t_sd.is_contiguous():       # cuDNN returns BSHD: a row-major [T, D] matrix
                K.note()
                _lib.check(_lib.lib().rrfp_copy_rows(
                    C.c_void_p(d_qkv.data_ptr() + i * D * 2), C.c_longlong(d_qkv.stride(0) * 2),
                    C.c_void_p(t.data_ptr()), C.c_longlong(D * 2), T, C.c_longlong(D * 2), K._stream()))
            else:
                d_qkv[:, i * D:(i + 1) * D].view(T, H, Dh).copy_(t_sd)

    def backward_weight(self, mb: int):
        """W task (decomposed backward): the FC1/FC2 weight gradients (plus LM
        head / projector / prologue) from the saved dy and d_pre, and the LN1 /
        LN2 parameter gradients from the saved LayerNorm input gradients (off the
        B-input chain, where nothing overlapped them); the attention weight
        gradients were done in B (see backward_input).  Layers alternate
        between the main and the side stream (independent GEMMs fill each
        other's tail waves); joined at the end."""
        if not self.decompose:
            return
        cfg = self.cfg
        S, D, Fd, Dl = cfg.seq, cfg.d_model, self.Fl, self.Dl
        T = self.rows[mb]
        main = torch.cuda.current_stream()
        side = self.side or main
        fork = torch.cuda.Event()
        fork.record(main)
        side.wait_event(fork)
        for li in reversed(range(len(self.layers))):
            g = self.g[li]
            # the last layer's output gradient is the B mailbox slot itself (interior stages)
            gy = (self.bwd_in[mb][:T] if li == len(self.layers) - 1 and self.epilogue is None
                  else self.gy[mb, li, :T])
            gpre = self.gpre[mb, li, :T]
            part = self.parts[li]
            with torch.cuda.stream(side if li % 2 else main):
                # LayerNorm parameter gradients (memory-bound: they overlap the other stream's GEMMs)
                lnb = _ln_bwd_fused if self.ln_fused else _ln_bwd
                if part != "attn":
                    x2 = self._layer_input(mb, li) if part == "mlp" else self.x2[mb, li, :T]
                    if self.ln_fused:   # + b_2's gradient (column sum of gy) in the same pass
                        _ln_bwd_fused(self.gln2[mb, li, :T], x2, self.m2[mb, li, :T], self.r2[mb, li, :T], None,
                                      gy, None, g["ln2_g"], g["ln2_b"], g["b_2"])
                    else:
                        _ln_bwd(self.gln2[mb, li, :T], x2, self.m2[mb, li, :T], self.r2[mb, li, :T], None,
                                None, None, g["ln2_g"], g["ln2_b"])
                if part != "mlp":
                    lnb(self.gln1[mb, li, :T], self._layer_input(mb, li), self.m1[mb, li, :T],
                        self.r1[mb, li, :T], None, None, None, g["ln1_g"], g["ln1_b"])
                if part != "attn":
                    K.gemm(gy, self.act[mb, li, :T], g["w_2"], epi=K.EPI_ACC_F32, a_mn=True,
                           b_mn=True, accumulate=True, m=D, n=Fd, k=T)
                    if not self.ln_fused:
                        _bias_grad(gy, g["b_2"])
                    K.gemm(gpre, self.h2[mb, li, :T], g["w_1"], epi=K.EPI_ACC_F32, a_mn=True,
                           b_mn=True, accumulate=True, m=Fd, n=D, k=T)
                    if not self.colsum_epi:   # (else reduced by B's FC2-dgrad epilogue)
                        _bias_grad(gpre, g["b_1"])
                if self.w_split == "all" and part != "mlp":
                    gx2, gqkv = self.gx2[mb, li, :T], self.gqkv[mb, li, :T]
                    K.gemm(gx2, self.o_view[mb][li], g["w_o"], epi=K.EPI_ACC_F32, a_mn=True,
                           b_mn=True, accumulate=True, m=D, n=Dl, k=T)
                    _bias_grad(gx2, g["b_o"])
                    K.gemm(gqkv, self.h1[mb, li, :T], g["w_qkv"], epi=K.EPI_ACC_F32, a_mn=True,
                           b_mn=True, accumulate=True, m=3 * Dl, n=D, k=T)
                    _bias_grad(gqkv, g["b_qkv"])
        with torch.cuda.stream(side):
            if self.last:
                K.gemm(self.logits[mb], self.hf[mb], self.g_head["w_lm"], epi=K.EPI_ACC_F32, a_mn=True,
                       b_mn=True, accumulate=True, m=cfg.vocab, n=D, k=S)
            if self.epilogue == "projector":
                dyp = self.bwd_in[mb][:T]
                K.gemm(dyp, self.y[mb, len(self.layers) - 1, :T], self.g_proj["w_proj"], epi=K.EPI_ACC_F32,
                       a_mn=True, b_mn=True, accumulate=True, m=dyp.shape[1], n=D, k=T)
                _bias_grad(dyp, self.g_proj["b_proj"])
            if self.prologue:
                self._prologue_wgrad(mb, self.gx0[mb, :T])
        join = torch.cuda.Event()
        join.record(side)
        main.wait_event(join)

    def release(self):
        """Drop every device buffer and captured graph now (a pipeline's stages
        hold ~100 GB at PP=1; bench builds several pipelines in one process)."""
        self.graphs.clear()
        self.attn_aux = self.o_view = None
        for k in list(vars(self)):
            if isinstance(getattr(self, k), (torch.Tensor, list, dict)) and k not in ("layers", "rows", "T_v"):
                setattr(self, k, None)

    def zero_grads(self):
        self.grad_flat.zero_()
        if self.last:
            self.loss.zero_()

    # ----------------------------------------------------------- capture
    def run_task(self, kind: str, mb: int):
        # GEMM grids of this stage's bodies are fixed at capture: an SM cap
        # (gemm_sm_cap) confines them to that many SMs (several stages sharing
        # one GPU as a PP emulation); 0 = the whole GPU
        L = _lib.lib()
        if self.gemm_sm_cap:
            L.rrfp_gemm_reserve_sms(max(0, torch.cuda.get_device_properties(self.device).multi_processor_count
                                        - self.gemm_sm_cap))
        try:
            if kind == "F":
                self.forward(mb)
            elif kind == "B":
                self.backward_input(mb)
            else:
                self.backward_weight(mb)
        finally:
            if self.gemm_sm_cap:
                L.rrfp_gemm_reserve_sms(0)

    def warmup(self, stream=None):
        """Run every body once eagerly (cuDNN plan selection, module loads,
        GEMM workspaces) on the capture stream; no host synchronisation, so
        the ranks of a TP group can warm up concurrently (their all-reduces
        wait for each other on the device).  Returns the stream."""
        stream = stream or torch.cuda.Stream(self.device)
        stream.wait_stream(torch.cuda.current_stream(self.device))   # parameter / data init
        with torch.cuda.stream(stream):
            for mb in range(self.M):
                for kind in ("F", "B", "W") if self.decompose else ("F", "B"):
                    self.run_task(kind, mb)
        self._cap_stream = stream
        return stream

    def capture(self):
        """One CUDA graph per (kind, mb) (after warmup() and a synchronize);
        returns 3*M raw cudaGraph_t handles indexed kind*M + mb with kind
        B=0, F=1, W=2 (None where no work)."""
        # F is captured before B/W: the B graph must bind the attention outputs
        # (o, lse) that the CAPTURED F graph writes, not the warm-up's.
        kinds = ["F", "B", "W"] if self.decompose else ["F", "B"]
        stream = self._cap_stream
        self.zero_grads()
        raw = [None] * (3 * self.M)
        for kind in kinds:
            ki = {"B": 0, "F": 1, "W": 2}[kind]
            for mb in range(self.M):
                g = torch.cuda.CUDAGraph(keep_graph=True)
                before = K.LAUNCHES[0]
                with torch.cuda.graph(g, stream=stream):
                    self.run_task(kind, mb)
                self.kernel_counts[(kind, mb)] = K.LAUNCHES[0] - before
                self.graphs[(kind, mb)] = g
                raw[ki * self.M + mb] = g.raw_cuda_graph()
        torch.cuda.synchronize(self.device)
        return raw

    def capture_bodies(self, stream=None):
        """warmup() + synchronize + capture() for a stage without TP peers."""
        stream = self.warmup(stream)
        stream.synchronize()
        return self.capture()
