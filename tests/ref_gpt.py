"""Plain PyTorch fp32 reference of the synthetic GPT (numerics oracle for the
floating-point stage compute): same weights (upcast), same tokens, no pipeline."""
import math

import torch
import torch.nn.functional as F


def ln(x, g, b, eps):
    return F.layer_norm(x, (x.shape[-1],), g, b, eps)


def reference_loss_and_grads(cfg, stages):
    """stages: list of StageCompute (any PP split).  Returns (loss, {name: grad})."""
    from paper_2605_18750_b200.model import init_layer_params
    params = {}
    for st in stages:
        for li, lid in enumerate(st.layers):
            # TP stages hold shards: rebuild the full layer from its deterministic init
            full = st.p[li] if st.R == 1 else init_layer_params(cfg, lid, st.device, st.model_seed)
            for k, v in full.items():
                params[f"L{lid}.{k}"] = v.float().clone().requires_grad_(True)
        if st.first:
            for k, v in st.emb.items():
                params[k] = v.float().clone().requires_grad_(True)
        if st.last:
            for k, v in st.head.items():
                params[k] = v.float().clone().requires_grad_(True)
    first, last = stages[0], stages[-1]
    M, S, D, H = first.M, cfg.seq, cfg.d_model, cfg.n_head
    Dh = D // H
    total = 0.0
    for mb in range(M):
        tok = first.tokens[mb].long()
        x = params["wte"][tok] + params["wpe"]
        for lid in range(cfg.n_layer):
            p = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"L{lid}.")}
            h = ln(x, p["ln1_g"], p["ln1_b"], cfg.eps)
            qkv = h @ p["w_qkv"].t() + p["b_qkv"]
            q, k, v = (qkv[:, i * D:(i + 1) * D].view(S, H, Dh).transpose(0, 1) for i in range(3))
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True, scale=1 / math.sqrt(Dh))
            o = o.transpose(0, 1).reshape(S, D)
            x2 = x + o @ p["w_o"].t() + p["b_o"]
            h2 = ln(x2, p["ln2_g"], p["ln2_b"], cfg.eps)
            a = F.gelu(h2 @ p["w_1"].t() + p["b_1"], approximate="tanh")
            x = x2 + a @ p["w_2"].t() + p["b_2"]
        hf = ln(x, params["lnf_g"], params["lnf_b"], cfg.eps)
        logits = hf @ params["w_lm"].t()
        total = total + F.cross_entropy(logits, last.targets[mb].long(), reduction="sum")
    loss = total / (M * S)
    loss.backward()
    return loss.item(), {k: v.grad for k, v in params.items()}


def device_grads(stages):
    out = {}
    for st in stages:
        for li, lid in enumerate(st.layers):
            for k, v in st.g[li].items():
                out[f"L{lid}.{k}"] = v
        if st.first:
            out.update(st.g_emb)
        if st.last:
            out.update(st.g_head)
    return out


def device_grads_tp(grid, cfg):
    """Full gradients from the TP shards of every stage (grid[s][r]): QKV / FC1
    rows and out-proj / FC2 columns concatenated in rank order; replicated
    parameters (LayerNorms, b_o, b_2, embedding, head) must agree across ranks
    (to fp32 atomic-order noise: their column reductions use atomics)."""
    out = {}
    D, R = cfg.d_model, len(grid[0])
    dl = D // R
    for row in grid:
        st0 = row[0]
        for li, lid in enumerate(st0.layers):
            gs = [st.g[li] for st in row]
            for k in gs[0]:
                if k in ("w_qkv", "b_qkv"):
                    parts = [torch.cat([g[k][i * dl:(i + 1) * dl] for g in gs]) for i in range(3)]
                    out[f"L{lid}.{k}"] = torch.cat(parts)
                elif k in ("w_1", "b_1"):
                    out[f"L{lid}.{k}"] = torch.cat([g[k] for g in gs])
                elif k in ("w_o", "w_2"):
                    out[f"L{lid}.{k}"] = torch.cat([g[k] for g in gs], dim=1)
                else:
                    for g in gs[1:]:
                        assert torch.allclose(g[k], gs[0][k], rtol=1e-3, atol=1e-6), \
                            f"replicated grad {k} differs across TP ranks"
                    out[f"L{lid}.{k}"] = gs[0][k]
        if st0.first:
            out.update(st0.g_emb)
        if st0.last:
            out.update(st0.g_head)
    return out


def compare(ref, got, cos_min=0.99, rel_max=0.05):
    bad = []
    for k, r in ref.items():
        g = got[k].float()
        cos = torch.nn.functional.cosine_similarity(r.flatten(), g.flatten(), dim=0).item()
        rel = ((r - g).norm() / (r.norm() + 1e-12)).item()
        if cos < cos_min or rel > rel_max:
            bad.append((k, round(cos, 4), round(rel, 4)))
    return bad


def _block(x, p, cfg, causal):
    T, D, H = x.shape[0], cfg.d_model, cfg.n_head
    Dh = D // H
    h = ln(x, p["ln1_g"], p["ln1_b"], cfg.eps)
    qkv = h @ p["w_qkv"].t() + p["b_qkv"]
    q, k, v = (qkv[:, i * D:(i + 1) * D].view(T, H, Dh).transpose(0, 1) for i in range(3))
    o = F.scaled_dot_product_attention(q, k, v, is_causal=causal, scale=1 / math.sqrt(Dh))
    o = o.transpose(0, 1).reshape(T, D)
    x2 = x + o @ p["w_o"].t() + p["b_o"]
    h2 = ln(x2, p["ln2_g"], p["ln2_b"], cfg.eps)
    a = F.gelu(h2 @ p["w_1"].t() + p["b_1"], approximate="tanh")
    return x2 + a @ p["w_2"].t() + p["b_2"]


def _prefix(st):
    return "V" if st.part == "vit" else "L"


def reference_mm_loss_and_grads(spec, stages):
    """Config 4 reference: ViT on each microbatch's T_v patch rows -> projector ->
    [visual rows, text embeddings] -> causal GPT -> loss over all positions."""
    params = {}
    for st in stages:
        for li, lid in enumerate(st.layers):
            for k, v in st.p[li].items():
                params[f"{_prefix(st)}{lid}.{k}"] = v.float().clone().requires_grad_(True)
        for d in (st.emb, st.head, st.pe, st.proj):
            if d:
                for k, v in d.items():
                    params[k] = v.float().clone().requires_grad_(True)
    vit0 = [st for st in stages if st.prologue == "patches"][0]
    llm0 = [st for st in stages if st.prologue == "merge"][0]
    last = stages[-1]
    vc, lc = spec.vit, spec.llm
    M, S = vit0.M, lc.seq
    total = 0.0
    for mb in range(M):
        T = vit0.rows[mb]
        x = vit0.patches[mb, :T].float() @ params["w_pe"].t() + params["b_pe"]
        for lid in range(vc.n_layer):
            p = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"V{lid}.")}
            x = _block(x, p, vc, False)
        vis = x @ params["w_proj"].t() + params["b_proj"]
        tok = llm0.tokens[mb, T:].long()
        text = params["wte"][tok] + params["wpe"][T:S]
        x = torch.cat([vis, text])
        for lid in range(lc.n_layer):
            p = {k.split(".", 1)[1]: v for k, v in params.items() if k.startswith(f"L{lid}.")}
            x = _block(x, p, lc, True)
        hf = ln(x, params["lnf_g"], params["lnf_b"], lc.eps)
        logits = hf @ params["w_lm"].t()
        total = total + F.cross_entropy(logits, last.targets[mb].long(), reduction="sum")
    loss = total / (M * S)
    loss.backward()
    return loss.item(), {k: v.grad for k, v in params.items()}


def device_grads_mm(stages):
    out = {}
    for st in stages:
        for li, lid in enumerate(st.layers):
            for k, v in st.g[li].items():
                out[f"{_prefix(st)}{lid}.{k}"] = v
        for d in (st.g_emb, st.g_head, st.g_pe, st.g_proj):
            if d:
                out.update(d)
    return out
