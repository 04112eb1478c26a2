"""GPT stage compute through the device pipeline vs a torch fp32 reference.

Tolerance (bf16 activations, fp32 accumulation; accumulation ORDER differs
between schedules): |loss - ref| / ref <= 1e-2 and per-tensor gradient
cosine >= 0.99 with relative L2 error <= 5%.
"""
import pytest
import torch

from ref_gpt import compare, device_grads, reference_loss_and_grads

pytestmark = pytest.mark.gpu

SMALL = dict(n_layer=4, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=256)


def _cfg():
    from paper_2605_18750_b200.model import GPTConfig
    return GPTConfig(**SMALL)


def test_eager_single_stage_matches_fp32_reference():
    from paper_2605_18750_b200.model import StageCompute
    cfg = _cfg()
    st = StageCompute(cfg, 0, 1, 3, "cuda")
    st.zero_grads()
    for mb in range(3):
        st.forward(mb)
        st.backward_input(mb)
    torch.cuda.synchronize()
    loss = (st.loss.sum() / (cfg.seq * 3)).item()
    ref_loss, ref_grads = reference_loss_and_grads(cfg, [st])
    assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
    assert not compare(ref_grads, device_grads([st]))


@pytest.mark.parametrize("n_stages,hint,mode,head_cost,w_split,split", [
    (1, "bf", "free", 0, "fc", "layer"), (2, "bf", "free", 0, "fc", "layer"),
    (4, "bfw", "free", 0, "fc", "layer"), (2, "bf", "fixed", 0, "fc", "layer"),
    (4, "bf", "replay", 0, "fc", "layer"), (2, "bfw", "free", 1.4, "fc", "layer"),
    (2, "bfw", "free", 0, "all", "layer"),
    # stage boundaries inside layers (attention half | MLP half)
    (3, "bf", "free", 1.4, "fc", "half"), (3, "bfw", "free", 1.4, "fc", "half"),
    (3, "bfw", "free", 0, "all", "half"), (5, "bf", "fixed", 1.4, "fc", "half")])
def test_pipeline_iteration_matches_fp32_reference(n_stages, hint, mode, head_cost, w_split, split):
    from paper_2605_18750_b200.pipeline import GpuPipeline
    cfg = _cfg()
    pipe = GpuPipeline(cfg, n_stages, 4, hint=hint, mode=mode, head_cost=head_cost, w_split=w_split,
                       split=split)
    if head_cost and split == "layer":
        assert [len(st.layers) for st in pipe.stages] == [3, 1]   # balanced against the LM head
    if split == "half":   # some stage starts with an MLP half and some ends with an attention half
        assert any(st.parts[0] == "mlp" for st in pipe.stages)
        assert any(st.parts[-1] == "attn" for st in pipe.stages)
    try:
        for _ in range(2):        # graphs replay: the second iteration must match too
            loss = pipe.step(watchdog_secs=60).item()
        tr, met = pipe.trace()
        assert len(tr.execs()) == pipe.workload.task_count()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()


@pytest.mark.parametrize("n_stages,tp,hint,mode,split", [
    (1, 2, "bf", "free", "layer"), (2, 2, "bf", "free", "layer"), (2, 2, "bfw", "free", "layer"),
    (2, 2, "bf", "fixed", "layer"), (3, 2, "bfw", "free", "half")])
def test_tp_pipeline_matches_fp32_reference(n_stages, tp, hint, mode, split):
    """Config 3 on one GPU: TP=2 lanes per stage, column/row-parallel GEMMs and
    the peer-memory all-reduce kernel; loss and (unsharded) gradients against
    the non-parallel fp32 reference; replicated gradients bit-identical across ranks."""
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from ref_gpt import device_grads_tp
    cfg = _cfg()
    pipe = GpuPipeline(cfg, n_stages, 4, hint=hint, mode=mode, tp_size=tp, split=split)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        for row in pipe.grid:
            for st in row:
                assert st.tp.error() == 0
        assert torch.equal(pipe.grid[-1][0].loss, pipe.grid[-1][1].loss)   # ranks agree bit-exactly
        tr, met = pipe.trace()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads_tp(pipe.grid, cfg))
        assert not bad, bad[:5]
    finally:
        pipe.close()


@pytest.mark.parametrize("n_stages,chunks,hint,mode,tp", [(2, 2, "bf", "free", 1), (2, 2, "bfw", "free", 1),
                                                          (2, 2, "bf", "replay", 1), (2, 2, "bf", "free", 2)])
def test_interleaved_chunks_match_fp32_reference(n_stages, chunks, hint, mode, tp):
    """C=2 virtual stages per lane (chunk-wrap edge N-1 -> 0),
    GPT bodies selected per (kind, chunk, mb) by the device dispatcher."""
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from ref_gpt import device_grads_tp
    cfg = _cfg()
    pipe = GpuPipeline(cfg, n_stages, 4, hint=hint, mode=mode, n_chunks=chunks, tp_size=tp)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        tr, met = pipe.trace()
        assert len(tr.execs()) == pipe.workload.task_count() * tp
        assert {e.chunk for e in tr.execs()} == set(range(chunks))
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        got = device_grads_tp(pipe.grid, cfg) if tp > 1 else device_grads(pipe.stages)
        bad = compare(ref_grads, got)
        assert not bad, bad[:5]
    finally:
        pipe.close()


@pytest.mark.parametrize("n_stages,vit_stages,hint,mode", [(2, 1, "bf", "free"), (3, 2, "bfw", "free"),
                                                           (2, 1, "bf", "fixed")])
def test_multimodal_vit_llm_matches_fp32_reference(n_stages, vit_stages, hint, mode):
    """Config 4: ViT stages with per-microbatch visual-token counts (variable
    message rows, non-causal attention) -> projector -> LLM stages."""
    from paper_2605_18750_b200.model import GPTConfig, MultimodalSpec
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from ref_gpt import device_grads_mm, reference_mm_loss_and_grads
    vit = GPTConfig(n_layer=2, d_model=256, n_head=2, d_ff=512, vocab=0, seq=512, causal=False)
    llm = GPTConfig(n_layer=2, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=512)
    spec = MultimodalSpec(vit=vit, llm=llm, vit_stages=vit_stages, patch_tokens=128, d_patch=128,
                          max_images=4, image_seed=3)
    assert len(set(spec.visual_tokens(4))) > 1          # the microbatches really differ
    pipe = GpuPipeline(None, n_stages, 4, hint=hint, mode=mode, mm=spec)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        tr, met = pipe.trace()
        assert len(tr.execs()) == pipe.workload.task_count()
        ref_loss, ref_grads = reference_mm_loss_and_grads(spec, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads_mm(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()


def test_zb_h1_schedule_gpt_pipeline_matches_fp32_reference():
    """A ZB-H1-like FixedSchedule (W tasks deferred into the cool-down) driving
    the GPT bodies in FIXED mode on the device lanes."""
    import paper_2605_18750_b200 as P
    from paper_2605_18750_b200.pipeline import GpuPipeline, nominal_workload
    cfg = _cfg()
    sched = P.build_zb_h1_schedule(nominal_workload(cfg, 4, 4, True))
    pipe = GpuPipeline(cfg, 4, 4, hint="bfw", mode="fixed", schedule=sched)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        tr, met = pipe.trace()
        got = [[(e.direction, e.microbatch) for e in sorted(tr.execs(), key=lambda e: e.t_start)
                if e.stage == s] for s in range(4)]
        assert got == [[(t.direction, t.microbatch) for t in st] for st in sched.per_stage_order]
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()


def test_green_partition_pipeline_matches_fp32_reference():
    """The single-GPU pipeline emulation: each stage on its own SM partition
    (green context); numerics unchanged."""
    from paper_2605_18750_b200.pipeline import GpuPipeline
    cfg = _cfg()
    pipe = GpuPipeline(cfg, 4, 4, hint="bfw", green=True)
    try:
        assert pipe.green_sms >= 2
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()


@pytest.mark.parametrize("hint", ["bf", "bfw"])
def test_gpt_pp4_lane_decisions_match_oracle(hint):
    """GPT PP=4 with real bodies: every free-running arbitration (logged on the
    device) re-evaluates to the same decision under the reference's arbitrate;
    in replay mode the lanes' own decisions give run_rrfp's trace exactly."""
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from decision_check import check_decisions
    import paper_2605_18750_b200 as P
    import rrfp_oracle as O
    cfg = _cfg()
    pipe = GpuPipeline(cfg, 4, 8, hint=hint, mode="free", declog_cap=1024)
    try:
        for _ in range(2):
            pipe.step(watchdog_secs=60)
        log = pipe.decisions()
        assert sum(d["kind"] != "wait" for d in log) == pipe.workload.task_count()
        assert not check_decisions(log, pipe.workload, P.HintOrder(hint), 32)
    finally:
        pipe.close()
    pipe = GpuPipeline(cfg, 4, 8, hint=hint, mode="replay")
    try:
        pipe.step(watchdog_secs=60)
        tr, met = pipe.trace()
        ev, om = O.run_rrfp(O.from_workload_json(pipe.workload.to_json()), hint, 32, 0, "J0")
        got = sorted((e.t_start, e.t_end, e.stage, e.microbatch, e.direction) for e in tr.execs())
        want = sorted((a, b, s, mb, d) for (a, b, s, r, mb, c, d, k) in ev if k == "exec")
        assert got == want
        assert met.makespan == om["makespan"]
    finally:
        pipe.close()


# ---------------------------------------------------------------------------
# numerics at the benchmarked shapes: the GPT-1.3B layer
# (d 2048, S 2048, 16 heads, ffn 8192, V 50304) and the 7B TP=2 layer (d 4096,
# 32 heads, ffn 16384), two layers, two microbatches, same tolerances as above.
GPT13B_SLICE = dict(n_layer=2, d_model=2048, n_head=16, d_ff=8192, vocab=50304, seq=2048)
GPT7B_SLICE = dict(n_layer=2, d_model=4096, n_head=32, d_ff=16384, vocab=50304, seq=2048)


@pytest.mark.parametrize("hint,mode", [("bf", "free"), ("bfw", "free"), ("bf", "fixed")])
def test_gpt13b_slice_pp2_matches_fp32_reference(hint, mode):
    """PP=2 with one 1.3B layer per stage; mode "fixed" + hint bf is the 1F1B run."""
    from paper_2605_18750_b200.model import GPTConfig
    from paper_2605_18750_b200.pipeline import GpuPipeline
    cfg = GPTConfig(**GPT13B_SLICE)
    pipe = GpuPipeline(cfg, 2, 2, hint=hint, mode=mode)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=120).item()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()
    torch.cuda.empty_cache()


def test_gpt7b_slice_tp2_matches_fp32_reference():
    """Config 3's layer at TP=2 x PP=1 (two lanes on one GPU, peer-memory all-reduce)."""
    from paper_2605_18750_b200.model import GPTConfig
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from ref_gpt import device_grads_tp
    cfg = GPTConfig(**GPT7B_SLICE)
    pipe = GpuPipeline(cfg, 1, 2, hint="bf", mode="free", tp_size=2)
    try:
        for _ in range(2):
            loss = pipe.step(watchdog_secs=120).item()
        for row in pipe.grid:
            for st in row:
                assert st.tp.error() == 0
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads_tp(pipe.grid, cfg))
        assert not bad, bad[:5]
    finally:
        pipe.close()
    torch.cuda.empty_cache()


def test_pipeline_with_own_attention_backward(monkeypatch):
    """RRFP_ATTN_BWD=own: the tcgen05 attention backward inside the captured bodies."""
    monkeypatch.setenv("RRFP_ATTN_BWD", "own")
    from paper_2605_18750_b200.pipeline import GpuPipeline
    cfg = _cfg()
    pipe = GpuPipeline(cfg, 2, 4, hint="bfw", mode="free")
    try:
        assert all(st.own_attn_bwd for st in pipe.stages)
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()


@pytest.mark.parametrize("hint", ["bf", "bfw"])
def test_pipeline_with_opt_in_fusions(monkeypatch, hint):
    """The opt-in fusions inside the captured bodies: the one-pass LayerNorm
    reductions (RRFP_LN_FUSED=1: LN parameter + adjacent bias gradients) and the
    FC1 bias gradient in the FC2-dgrad epilogue (RRFP_COLSUM_EPI=1), fused B and
    BFW; the default LM-head statistics epilogue is on in both."""
    monkeypatch.setenv("RRFP_LN_FUSED", "1")
    monkeypatch.setenv("RRFP_COLSUM_EPI", "1")
    from paper_2605_18750_b200.pipeline import GpuPipeline
    cfg = _cfg()
    pipe = GpuPipeline(cfg, 2, 4, hint=hint, mode="free")
    try:
        assert all(st.ln_fused and st.colsum_epi for st in pipe.stages)
        assert pipe.stages[-1].ce_fused
        for _ in range(2):
            loss = pipe.step(watchdog_secs=60).item()
        ref_loss, ref_grads = reference_loss_and_grads(cfg, pipe.stages)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (loss, ref_loss)
        bad = compare(ref_grads, device_grads(pipe.stages))
        assert not bad, bad[:5]
    finally:
        pipe.close()
