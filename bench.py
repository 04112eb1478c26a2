"""Benchmark: readiness-driven pipeline iteration of synthetic GPT-1.3B on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--hint bf|bfw|1f1b] [--mb 32] [--jitter J0..J3] [--layers 24]

N=1 runs PP=1 (the single-GPU configuration of BASELINE.json configs[1]);
``--gpus N`` > 1 runs PP=N (N/tp stages x tp ranks), one process per GPU: under
torchrun as launched by the driver, or -- started as plain ``python bench.py
--gpus N`` -- by re-executing itself under ``torch.distributed.run`` with N
ranks (mailboxes over CUDA IPC / NVLink).  A step = one training iteration over
M=32 microbatches (F + B (+W) for every microbatch, fp32 weight-gradient
accumulation), launched as ONE graph per stage whose device dispatcher picks
every task.  Prints one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os

# before any CUDA context exists: one hardware queue per stream, so a lane's
# spinning dispatcher never serialises another stream's work (as the package sets)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "iter/s & tokens/s at PP=2/4/8 under jitter vs fixed-order 1F1B; bubble %"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TASK_TIMES = os.path.join(ROOT, "profiles", "task_times_gpt1p3b.json")


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p["bf16_tflops_sustained"], p["bf16_tflops"], p["hbm_gbs"], "measured"
    except Exception:
        return 1400.0, 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = sorted(int(r[0]) for r in self.rows if r and r[0].isdigit())
        mx = max((int(r[1]) for r in self.rows if len(r) > 1 and r[1].isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU runtime (live.run_live restated in oracle/) on this
    host, executing the same iteration's task graph with the per-task
    durations our kernels take on the B200 (profiles/task_times_gpt1p3b.json)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.hint == "1f1b":
        # the reference's only wall-clock executor (live.run_live) is readiness-
        # driven; 1F1B exists only on its virtual clock (baselines.run_fixed)
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no wall-clock 1F1B "
                          "executor (live.run_live arbitrates; 1F1B is baselines.run_fixed, virtual)"}),
              flush=True)
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rrfp_oracle as O
    n = max(1, args.gpus // args.tp)
    times = default_task_times(n, model_config(args).n_layer)
    lat = {}
    dec = args.hint == "bfw"
    for s in range(n):
        for mb in range(args.mb):
            lat[("F", s, mb, 0)] = int(times["F"][s])
            if dec:
                lat[("B", s, mb, 0)] = int(times["Bin"][s])
                lat[("W", s, mb, 0)] = int(times["W"][s])
            else:
                lat[("B", s, mb, 0)] = int(times["B"][s])
    w = {"N": n, "M": args.mb, "C": 1, "R": 1, "lat": lat, "comm": {"kind": "constant", "value": 0},
         "dec": dec, "beta": 0.5}
    hint = "bf" if args.hint == "1f1b" else args.hint
    for _ in range(args.warmup):
        O.run_live(w, hint, 32, 1.0, seed=0, jitter=args.jitter)
    t0 = time.perf_counter()
    mks = []
    for _ in range(args.steps):
        _, mk = O.run_live(w, hint, 32, 1.0, seed=0, jitter=args.jitter)
        mks.append(mk)
    dt = (time.perf_counter() - t0) / args.steps
    v = 1.0 / dt
    cores = 3 * n     # threads run_live uses (sender / receiver / worker per stage); GIL-bound
    line = {"metric": METRIC, "value": round(v, 4), "unit": "iter/s", "impl": "reference",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "tokens_per_s": round(v * args.mb * 2048, 1),
            "config": workload_config(args, n),
            "cpu_baseline": {"value": round(v, 4), "unit": "iter/s", "cores": cores, "kind": "port",
                             "os_cpu_count": os.cpu_count(), "sched_affinity": len(os.sched_getaffinity(0)),
                             "sample": f"oracle.run_live: {3 * n} threads (GIL-bound; host has "
                                       f"{len(os.sched_getaffinity(0))} cores), {n}x{args.mb} tasks, "
                                       f"task durations = B200-measured GPT-1.3B per-task times "
                                       f"(profiles/task_times_gpt1p3b.json, this bench's kernels); what "
                                       f"differs from our arm is the runtime: Python threads + queues vs "
                                       f"device lanes"},
            "e2e": {"value": round(v, 4), "unit": "iter/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def default_task_times(n_stages, n_layer=24):
    """Per-stage F/B/Bin/W task times (µs) of GPT-1.3B on B200, measured by
    this bench (profiles/task_times_gpt1p3b.json) or estimated before that."""
    try:
        with open(TASK_TIMES) as f:
            t = json.load(f)
        row = t.get(str(n_stages))
        if row:
            return row
    except Exception:
        pass
    per_layer_f = 260.0
    lp = n_layer / n_stages
    f = [per_layer_f * lp for _ in range(n_stages)]
    f[-1] += 500.0
    return {"F": f, "B": [2.1 * x for x in f], "Bin": [1.15 * x for x in f], "W": [0.95 * x for x in f]}


def model_config(args):
    """GPT-1.3B (BASELINE config 2), GPT-7B (config 3, run with --tp 2) or, for
    --model mm, the LLM part (7B) of config 4."""
    from paper_2605_18750_b200.model import GPTConfig
    if args.model in ("7b", "mm"):
        return GPTConfig(n_layer=args.layers or 32, d_model=4096, n_head=32, d_ff=16384)
    return GPTConfig(n_layer=args.layers or 24)


def mm_spec(args):
    """Config 4: ViT-H/14 (32 layers, d=1280, 256 tokens/image, 1..8 images per
    microbatch, seeded) on stage 0 + the 7B LLM on the remaining stages."""
    if args.model != "mm":
        return None
    from paper_2605_18750_b200.model import VIT_H14, MultimodalSpec
    return MultimodalSpec(vit=VIT_H14, llm=model_config(args), vit_stages=1)


def iteration_flops(args, cfg):
    """Useful matmul FLOPs of one iteration (F + B-input + W of every layer and the LM head)."""
    fF, fB, fW = cfg.flops_per_layer()
    total = args.mb * (cfg.n_layer * (fF + fB + fW) + 3 * cfg.flops_head())
    spec = mm_spec(args)
    if spec is not None:
        for t in spec.visual_tokens(args.mb):
            vF, vB, vW = spec.vit.flops_per_layer(t)
            total += spec.vit.n_layer * (vF + vB + vW) + 3 * 2 * t * spec.vit.d_model * (spec.d_patch + spec.llm.d_model)
    return total


def workload_config(args, n):
    from paper_2605_18750_b200.model import split_units
    c = model_config(args)
    if args.model == "mm":
        return {"workload": f"config 4: ViT-H/14 (32 L, d=1280, 256 tok/image, 1..8 images/mb seeded) on stage 0 "
                            f"+ GPT-7B (L={c.n_layer}) on stages 1..{n - 1}, s={c.seq}, M={args.mb}",
                "model": "vit-h14+gpt-7b-synthetic", "global_batch": args.mb, "seq_len": c.seq,
                "parallelism": f"pp{n}", "hint": args.hint, "jitter": args.jitter, "buffer_limit": 32,
                "l2": "inputs larger than L2 (activations >> 126 MB per step)"}
    par = f"pp{n}" + (f"xtp{args.tp}" if args.tp > 1 else "") + (f"xc{args.chunks}" if args.chunks > 1 else "")
    return {"workload": f"GPT-{args.model.upper()} synthetic (L={c.n_layer}, d={c.d_model}, h={c.n_head}, "
                        f"ffn={c.d_ff}, V={c.vocab}, s={c.seq}, mbs=1), PP={n}, TP={args.tp}, C={args.chunks}, M={args.mb}",
            "model": f"gpt-{args.model}-synthetic", "global_batch": args.mb, "seq_len": c.seq,
            "parallelism": par, "hint": args.hint, "jitter": args.jitter,
            "layer_split": [[f"{l}{pt[0] if pt != 'full' else ''}" for l, pt in
                             split_units(c.n_layer, n * args.chunks, s_, args.head_cost if args.chunks == 1 else 0,
                                         stage_split(args))] for s_ in range(n * args.chunks)]
                           if n * args.chunks > 1 else [c.n_layer],
            "buffer_limit": 32, "l2": "inputs larger than L2 (activations >> 126 MB per step)"}


# ------------------------------------------------------------------ our arm
def roofline_gemm_calls(cfg):
    """One layer's twelve F/B/W GEMMs, shapes and epilogues exactly as the stage
    bodies issue them: [(fn, flops), ...] (also used by tools/prof_gemm.py)."""
    import torch
    from paper_2605_18750_b200 import kernels as K
    S, D, Fd = cfg.seq, cfg.d_model, cfg.d_ff
    bf = torch.bfloat16
    dev = "cuda"
    x, w_qkv, w_o, w_1, w_2 = (torch.randn(S, D, device=dev).to(bf), torch.randn(3 * D, D, device=dev).to(bf),
                               torch.randn(D, D, device=dev).to(bf), torch.randn(Fd, D, device=dev).to(bf),
                               torch.randn(D, Fd, device=dev).to(bf))
    bias = torch.zeros(Fd, device=dev).to(bf)
    qkv, y, pre, act = (torch.empty(S, 3 * D, device=dev, dtype=bf), torch.empty(S, D, device=dev, dtype=bf),
                        torch.empty(S, Fd, device=dev, dtype=bf), torch.empty(S, Fd, device=dev, dtype=bf))
    gq, g1, g2 = torch.zeros(3 * D, D, device=dev), torch.zeros(Fd, D, device=dev), torch.zeros(D, Fd, device=dev)
    go, dx = torch.zeros(D, D, device=dev), torch.empty(S, D, device=dev, dtype=bf)
    return [
        (lambda: K.gemm(x, w_qkv, qkv, bias=bias[:3 * D]), 2 * S * D * 3 * D),
        (lambda: K.gemm(x, w_o, y, epi=K.EPI_RESID, bias=bias[:D], r=x), 2 * S * D * D),
        (lambda: K.gemm(x, w_1, pre, epi=K.EPI_BIAS_GELU, c2=act, bias=bias), 2 * S * D * Fd),
        (lambda: K.gemm(act, w_2, y, epi=K.EPI_RESID, bias=bias[:D], r=x), 2 * S * D * Fd),
        (lambda: K.gemm(x, w_2, pre, epi=K.EPI_GELU_BWD, b_mn=True, r=pre), 2 * S * D * Fd),
        (lambda: K.gemm(pre, w_1, y, b_mn=True), 2 * S * D * Fd),
        (lambda: K.gemm(qkv, w_qkv, y, b_mn=True), 2 * S * D * 3 * D),
        (lambda: K.gemm(x, act, g2, epi=K.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True), 2 * S * D * Fd),
        (lambda: K.gemm(pre, x, g1, epi=K.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True), 2 * S * D * Fd),
        (lambda: K.gemm(qkv, x, gq, epi=K.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True), 2 * S * D * 3 * D),
        # attention out-projection backward: dgrad dY.W_o and wgrad dY^T.O (the 2048^3 shapes)
        (lambda: K.gemm(y, w_o, dx, b_mn=True), 2 * S * D * D),
        (lambda: K.gemm(y, x, go, epi=K.EPI_ACC_F32, a_mn=True, b_mn=True, accumulate=True), 2 * S * D * D),
    ]


def gemm_roofline(cfg, peak_tf):
    """Time the dominant kernel (the stage GEMMs) with CUDA events on its own
    launch stream, shapes and epilogues exactly as one layer's F/B/W issue them.
    Timed alone (10 back-to-back reps), so ``peak_tf`` is the BURST peak."""
    import torch
    calls = roofline_gemm_calls(cfg)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())   # operands initialised on the current stream
    with torch.cuda.stream(st):
        for fn, _ in calls:
            fn()
        st.synchronize()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            for fn, _ in calls:
                fn()
        e1.record(st)
        st.synchronize()
    ms = e0.elapsed_time(e1) / (reps * len(calls))
    flops = sum(f for _, f in calls) / len(calls)
    achieved = flops / (ms * 1e-3) / 1e12
    # per shape (each GEMM alone, same stream): the small 2048^3 ones are the weak spot
    per = []
    with torch.cuda.stream(st):
        for fn, f in calls:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(5):
                fn()
            b.record(st)
            st.synchronize()
            per.append(round(f / (a.elapsed_time(b) / 5 * 1e-3) / 1e12, 1))
    # the same twelve M/N/K and operand layouts through cuBLAS (torch.mm, bf16 out, no
    # fused epilogue): the library reference point under the same clocks
    cub = []
    try:
        S, D, Fd = cfg.seq, cfg.d_model, cfg.d_ff
        bf = torch.bfloat16
        mk = lambda r, c: torch.randn(r, c, device="cuda").to(bf)
        x, w_qkv, w_o, w_1, w_2 = mk(S, D), mk(3 * D, D), mk(D, D), mk(Fd, D), mk(D, Fd)
        pre, qkv = mk(S, Fd), mk(S, 3 * D)
        shapes = [lambda: torch.mm(x, w_qkv.t()), lambda: torch.mm(x, w_o.t()), lambda: torch.mm(x, w_1.t()),
                  lambda: torch.mm(pre, w_2.t()), lambda: torch.mm(x, w_2), lambda: torch.mm(pre, w_1),
                  lambda: torch.mm(qkv, w_qkv), lambda: torch.mm(x.t(), pre), lambda: torch.mm(pre.t(), x),
                  lambda: torch.mm(qkv.t(), x), lambda: torch.mm(x, w_o), lambda: torch.mm(x.t(), x)]
        with torch.cuda.stream(st):
            for fn in shapes:
                fn()
            tot = 0.0
            for fn, (_, f) in zip(shapes, calls):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(5):
                    fn()
                b.record(st)
                st.synchronize()
                t = a.elapsed_time(b) / 5 * 1e-3
                tot += t
                cub.append(round(f / t / 1e12, 1))
        cub_achieved = sum(f for _, f in calls) / tot / 1e12
    except Exception as e:
        cub_achieved = None
        cub = [repr(e)[:120]]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            traffic = json.load(f)["traffic_bytes_per_launch_mean"]
    except Exception:
        pass
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak_tf, "unit": "TFLOP/s",
            "frac": round(achieved / peak_tf, 3), "traffic": traffic,
            "traffic_unit": "bytes/launch (dram rd+wr, ncu --set full, profiles/gemm_traffic.json)",
            "kernel": "gemm_bf16_sm100_pair (cta_group::2 tcgen05.mma 256x256x16; clusters of two CTA pairs "
                      "sharing A by TMA multicast; half-width last wave; TMA 6-stage ring, TMEM x2, "
                      "TMA-store / reduce-add epilogue)",
            "per_launch": f"mean over one layer's 12 F/B/W GEMMs ({cfg.seq} tokens, d={cfg.d_model}, "
                          f"ffn={cfg.d_ff}); CUDA events on the launch stream, 10 reps, in this process "
                          "after the timed region (isolated: burst peak)",
            "per_gemm_tflops": per,
            "cublas_per_gemm_tflops": cub,
            "cublas_tflops": round(cub_achieved, 1) if cub_achieved else None,
            "cublas_note": "torch.mm on the same M/N/K and operand layouts, bf16 output, no fused epilogue "
                           "(library reference under the same clocks; ours also runs bias/GELU/residual/"
                           "f32-accumulate epilogues)",
            "share_of_step": "75.4% of device time (profiles/r02_bench_launches_summary_fused.txt, ncu launch list)",
            "avg_launch_us": round(ms * 1e3, 1)}


def _log(msg):
    sys.stderr.write(f"[bench {time.strftime('%H:%M:%S')}] {msg}\n")
    sys.stderr.flush()


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if os.environ.get("RRFP_SAME_DEVICE") == "1":     # 1-GPU test of the multi-process path
        local = 0
    torch.cuda.set_device(local)
    from paper_2605_18750_b200.jitter import PRESETS
    cfg = model_config(args)
    if world % args.tp:
        raise SystemExit(f"--tp {args.tp} must divide the number of processes {world}")
    n = world // args.tp if world > 1 else 1      # pipeline stages
    hint = "bf" if args.hint == "1f1b" else args.hint
    mode = "fixed" if args.hint == "1f1b" else "free"
    dist = None
    if world > 1:
        import torch.distributed as dist
        # plumbing only (handle exchange, barriers, max-over-ranks): gloo on host tensors
        dist.init_process_group("gloo")
    t_build = time.perf_counter()
    pipe, stages = build_pipe(cfg, args, hint, mode, world, PRESETS[args.jitter])
    t_build = time.perf_counter() - t_build
    _log(f"built in {t_build:.1f}s")
    clock_cal = None
    if dist:   # cross-GPU %globaltimer offsets, so the gathered trace is on one clock
        off, rtt = pipe.calibrate_clocks()
        allc = [None] * world
        dist.all_gather_object(allc, (off, rtt))
        clock_cal = {"offset_ns_vs_rank0": [c[0] for c in allc], "best_rtt_ns": [c[1] for c in allc]}
    # the step's input data held by this rank's stages (tokens / image patches /
    # targets): copied from pinned host memory every step of the e2e loop
    inputs = []
    for st in stages:
        for name in ("tokens", "patches", "targets"):
            t = getattr(st, name, None)
            if t is not None:
                inputs.append((t, t.cpu().pin_memory()))
    h2d = sum(h.numel() * h.element_size() for _, h in inputs)
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        pipe.step()
    barrier()
    _log("warm-up done")
    lane_stream = pipe.group.streams[next(iter(pipe.group.streams))]
    peak_sus, peak_burst, hbm, peak_kind = load_peaks()
    with ClockSampler(local) as clk:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lane_stream)
        for _ in range(args.steps):
            pipe.launch()
            pipe.wait()
        e1.record(lane_stream)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
        # end-to-end through the public API with host buffers
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for dev_t, host_t in inputs:
                dev_t.copy_(host_t, non_blocking=True)
            loss = pipe.step()
            if loss is not None:
                loss_h.copy_(loss.reshape(1), non_blocking=False)
        barrier()
        e2e_s = (time.perf_counter() - t0) / args.steps
    h2d_all = h2d
    if dist:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = t[0].item(), t[1].item()
        hb = torch.tensor([h2d], dtype=torch.int64)
        dist.all_reduce(hb)
        h2d_all = int(hb.item())
    _log("timed region done")
    tr, met = gather_trace(pipe, dist, world)
    from paper_2605_18750_b200.runtime import dispatch_latency
    bubble = met.bubble_fraction()
    it_s = 1000.0 / ms
    tok = args.mb * cfg.seq
    execs = tr.execs()
    task_us = {}
    for d in ("F", "B", "W"):
        per = []
        for s_ in range(n):
            xs = [e.t_end - e.t_start for e in execs if e.direction == d and e.stage == s_]
            per.append(round(sum(xs) / len(xs), 1) if xs else 0.0)
        task_us[d] = per
    roof = gemm_roofline(cfg, peak_burst)
    _log("roofline done")
    roof["peak_kind"] = f"bf16_tflops burst ({peak_kind}): the GEMMs are timed alone, back to back"
    roof["frac_vs_sustained"] = round(roof["achieved"] / peak_sus, 3)
    it_flops = iteration_flops(args, cfg)
    n_dev = max(1, world)
    act = cfg.seq * cfg.d_model * 2
    # per GPU: mailbox writes (F out + B out, to the same TP rank of the neighbour) and
    # TP all-reduce peer reads (4 per layer per microbatch, R-1 partials each)
    p2p = (2 * args.mb * act if n > 1 else 0) + \
        4 * (cfg.n_layer // n) * args.mb * act * (args.tp - 1)
    t_roof = it_flops / (n_dev * peak_sus * 1e12) + p2p / 770e9
    launches = pipe.kernel_launches_per_step() if hasattr(pipe, "kernel_launches_per_step") else 0
    if dist:
        lt = torch.tensor([launches], dtype=torch.int64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    line = {"metric": METRIC, "value": round(it_s, 4), "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, uniform tokens)",
            "config": workload_config(args, n),
            "tokens_per_s": round(it_s * tok, 1), "bubble_fraction": round(bubble, 4),
            "iteration_roofline": {"t_roof_ms": round(t_roof * 1e3, 2),
                                   "frac": round(t_roof * 1e3 / ms, 3),
                                   "definition": "sum stage FLOPs / (N_gpu * sustained bf16 peak) "
                                                 "+ per-GPU P2P + TP all-reduce bytes / 770 GB/s"},
            "roofline": roof,
            "task_us": task_us,
            "dispatch": dispatch_latency(tr, n),
            "e2e": {"value": round(1.0 / e2e_s, 4), "unit": "iter/s",
                    "h2d_bytes_per_step": int(h2d_all), "d2h_bytes_per_step": 4},
            "gpu_launches": int(launches) * args.steps,
            "gpu_launches_per_step": int(launches),
            "build_s": round(t_build, 1),
            "clock_calibration": clock_cal,
            "clocks": clk.summary()}
    # dispatcher profile: one more (untimed) iteration with lane_step_kernel's own
    # %globaltimer stamps (ncu cannot profile kernel nodes of conditional graphs)
    try:
        from paper_2605_18750_b200.runtime import dispatcher_profile
        pipe.group.enable_profile(16384)
        pipe.step()
        line["dispatch"]["step_kernel"] = dispatcher_profile(pipe.group.profile())
        pipe.group.enable_profile(0)
    except Exception as e:     # a profile must never cost the measurement
        line["dispatch"]["step_kernel"] = {"error": repr(e)[:200]}
    if rank == 0 and args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, n, task_us)
    if rank == 0 and args.model != "mm" and args.tp == 1 and args.chunks == 1:
        try:
            line["pipeline_model"] = pipeline_model(args, cfg, task_us, n)
        except Exception as e:   # a model table must never cost the measurement
            line["pipeline_model"] = {"error": repr(e)[:200]}
    if dist:
        line["p2p"] = p2p_block(pipe, cfg, args, dist, world, clock_cal)
    pipe.close()
    del pipe, stages, inputs
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    if args.emulate_pp > 1 and world == 1:
        # a fresh process: the PP=1 pipeline's ~110 GB must not share the GPU with it
        cmd = [sys.executable, os.path.abspath(__file__), "--emulate-only", "--emulate-pp", str(args.emulate_pp),
               "--w-split", args.w_split, "--split", args.split,
               *([] if args.green else ["--no-green"]),
               *(["--trace-dir", args.trace_dir] if args.trace_dir else []),
               "--steps", str(args.steps), "--warmup", str(args.warmup), "--mb", str(args.mb),
               "--sigmas", args.sigmas, "--compare-jitter", args.compare_jitter, "--comm-us", str(args.comm_us),
               "--head-cost", str(args.head_cost), "--model", args.model]
        if args.layers:
            cmd += ["--layers", str(args.layers)]
        p = subprocess.run(cmd, capture_output=True, text=True)
        sys.stderr.write(p.stderr[-4000:])
        lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
        line["emulated_pp"] = json.loads(lines[-1]) if (p.returncode == 0 and lines) else \
            {"error": f"rc={p.returncode}: {p.stderr[-300:]}"}
        # the smaller pipelines of the PP sweep (BASELINE metric: PP=2/4/8), J0 and the first
        # sigma only, one fresh process each
        extra = {}
        for n_pp in [int(x) for x in args.emulate_pp_extra.split(",") if x and int(x) != args.emulate_pp]:
            cmd2 = list(cmd)
            cmd2[cmd2.index("--emulate-pp") + 1] = str(n_pp)
            cmd2[cmd2.index("--compare-jitter") + 1] = args.compare_jitter.split(",")[0]
            p = subprocess.run(cmd2, capture_output=True, text=True)
            sys.stderr.write(p.stderr[-2000:])
            lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
            extra[f"pp{n_pp}"] = json.loads(lines[-1]) if (p.returncode == 0 and lines) else \
                {"error": f"rc={p.returncode}: {p.stderr[-300:]}"}
        if extra:
            line["emulated_pp_sweep"] = extra
    if args.compare or (world > 1 and args.compare is None):
        line["variants"] = compare_variants(cfg, args, world, dist, barrier)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def stage_split(args):
    """Stage boundaries at half-layers for the GPT pipeline (model.split_units); config 4 splits at layers."""
    return "layer" if args.model == "mm" else args.split


def build_pipe(cfg, args, hint, mode, world, jitter, comm_delay=None):
    if world > 1:
        from paper_2605_18750_b200.distributed import DistPipeline
        pipe = DistPipeline(cfg, args.mb, hint=hint, mode=mode, jitter=jitter, comm_delay=comm_delay,
                            tp_size=args.tp, n_chunks=args.chunks, mm=mm_spec(args), head_cost=args.head_cost,
                            w_split=args.w_split, split=stage_split(args))
        return pipe, pipe.vstages
    if args.model == "mm":
        raise SystemExit("--model mm (config 4) needs a pipeline of >= 2 GPUs")
    from paper_2605_18750_b200.pipeline import GpuPipeline
    pipe = GpuPipeline(cfg, 1, args.mb, hint=hint, mode=mode, jitter=jitter, comm_delay=comm_delay,
                       tp_size=args.tp, n_chunks=args.chunks, head_cost=args.head_cost, w_split=args.w_split)
    return pipe, pipe.stages


B_IN_FRAC, W_FRAC = 0.714, 0.307


def pipeline_model(args, cfg, task_us, n_meas, sigmas=(0.0, 0.5), pps=(2, 4, 8), device="cuda", grid=True,
                   grid_sigmas=(0.0, 0.1, 0.2, 0.3, 0.4, 0.5), grid_levels=("J0", "J1", "J2", "J3")):
    """Virtual-clock prediction of the PP sweep from THIS run's B200 task times
    (SURVEY 6.3 / 8d C5): per-layer F and B durations of the measured run,
    balanced layer split, LM head on the last stage, lognormal(0, sigma)
    compute factors per task (identical draws for every schedule) and
    lognormal(ln 100 us, sigma) per-edge comm delays.  1F1B = run_fixed, BF /
    BFW = run_rrfp, all in the device replay kernel.  A model, not a
    multi-GPU measurement: it says what the scheduler does with these kernels."""
    import math
    import numpy as np
    import paper_2605_18750_b200 as P
    from paper_2605_18750_b200.model import ATTN_FRAC, split_units
    from paper_2605_18750_b200.rng import substream
    L = cfg.n_layer

    def layer_eq(n, s_):   # the stage's layers in layer-equivalents (half-layers: ATTN_FRAC / 1 - ATTN_FRAC)
        w = {"full": 1.0, "attn": ATTN_FRAC, "mlp": 1.0 - ATTN_FRAC}
        return sum(w[pt] for _, pt in split_units(L, n, s_, args.head_cost, stage_split(args)))
    lay0 = [layer_eq(n_meas, s_) for s_ in range(n_meas)]
    # per-layer times from the measured first stage (no head), head from the last stage
    f_l = task_us["F"][0] / lay0[0]
    b_l = task_us["B"][0] / lay0[0]
    f_h = max(0.0, task_us["F"][-1] - f_l * lay0[-1]) if n_meas == 1 else task_us["F"][-1] - f_l * lay0[-1]
    b_h = max(0.0, task_us["B"][-1] - b_l * lay0[-1]) if n_meas == 1 else task_us["B"][-1] - b_l * lay0[-1]
    if n_meas == 1:   # the PP=1 stage holds every layer and the head: split by the measured ratio
        f_h, b_h = 1.6 * f_l, 1.27 * b_l
        f_l = task_us["F"][0] / (L + 1.6)
        b_l = task_us["B"][0] / (L + 1.27)
        f_h, b_h = 1.6 * f_l, 1.27 * b_l
    out = {"definition": pipeline_model.__doc__.split("\n\n")[0].strip().replace("\n", " "),
           "per_layer_us": {"F": round(f_l, 1), "B": round(b_l, 1)}, "head_us": {"F": round(f_h, 1), "B": round(b_h, 1)}}
    from paper_2605_18750_b200.jitter import PRESETS, build_injection_table

    def point(n, lay, sigma, jname, seed=0):
        res = {}
        for name in ("1f1b", "bf", "bfw"):
            dec = name == "bfw"
            lat = {}
            for s_ in range(n):
                for mb in range(args.mb):
                    x = float(np.exp(substream(11, "cjitter", s_, mb, "F").normal(0.0, sigma))) if sigma else 1.0
                    y = float(np.exp(substream(11, "cjitter", s_, mb, "B").normal(0.0, sigma))) if sigma else 1.0
                    fd = (f_l * lay[s_] + (f_h if s_ == n - 1 else 0)) * x
                    bd = (b_l * lay[s_] + (b_h if s_ == n - 1 else 0)) * y
                    lat[P.TaskId(s_, mb, 0, "F")] = max(1, int(fd))
                    if dec:
                        # B-input / W as fractions of the fused B (captured bodies of
                        # an interior stage, profiles/r01_task_times_ln_in_w.txt: 274 + 118 vs 384)
                        lat[P.TaskId(s_, mb, 0, "B")] = max(1, int(B_IN_FRAC * bd))
                        lat[P.TaskId(s_, mb, 0, "W")] = max(1, int(W_FRAC * bd))
                    else:
                        lat[P.TaskId(s_, mb, 0, "B")] = max(1, int(bd))
            comm = P.CommDelay()
            if sigma:
                comm = P.CommDelay(kind="lognormal", mu=math.log(args.comm_us), sigma=sigma, lo=0,
                                   hi=int(args.comm_us * 50), seed=17)
            w = P.Workload(num_stages=n, num_microbatches=args.mb, num_chunks=1, tp_group_size=1,
                           latency=lat, comm_delay=comm, decompose_backward=dec)
            jc = PRESETS[jname]
            if name == "1f1b":
                inj = build_injection_table(w, jc, seed) if jc.enabled else None
                tr, m = P.run_fixed(P.build_1f1b_schedule(w), w, injected_delays=inj, record_trace=False,
                                    device=device)
            else:
                tr, m = P.run_rrfp(w, name, 32, seed, jitter=jc, record_trace=False, device=device)
            res[name] = {"ms": round(m.makespan / 1e3, 2), "bubble": round(m.bubble_fraction(), 4)}
        for name in ("bf", "bfw"):
            res[name]["speedup_vs_1f1b"] = round(res["1f1b"]["ms"] / res[name]["ms"], 4)
        return res

    for n in pps:
        lay = [round(layer_eq(n, s_), 2) for s_ in range(n)]
        row = {"layers": lay}
        for sigma in sigmas:
            row[f"sigma{sigma}"] = point(n, lay, sigma, "J0")
        out[f"pp{n}"] = row
    if grid and 8 in pps:
        # the (sigma x J-preset) operating grid at PP=8 --
        # where does BFW / 1F1B reach the north star's 1.5x with these kernels?
        lay = out["pp8"]["layers"]
        g = {"sigmas": list(grid_sigmas), "levels": list(grid_levels), "bfw_speedup": {}, "bf_speedup": {},
             "bubble_1f1b": {}, "bubble_bfw": {}}
        for jname in grid_levels:
            for key in ("bfw_speedup", "bf_speedup", "bubble_1f1b", "bubble_bfw"):
                g[key][jname] = []
            for sigma in grid_sigmas:
                r = point(8, lay, sigma, jname)
                g["bfw_speedup"][jname].append(r["bfw"]["speedup_vs_1f1b"])
                g["bf_speedup"][jname].append(r["bf"]["speedup_vs_1f1b"])
                g["bubble_1f1b"][jname].append(r["1f1b"]["bubble"])
                g["bubble_bfw"][jname].append(r["bfw"]["bubble"])
        g["points_bfw_ge_1p5"] = [[j, sg] for j in grid_levels
                                  for sg, v in zip(grid_sigmas, g["bfw_speedup"][j]) if v >= 1.5]
        out["pp8_grid"] = g
    return out


def replay_prediction(pipe, name, sigma, nominal, floor_seed=11):
    """What the virtual-clock engine predicts for an emulated variant (ms):
    the device replay kernel on the variant's own workload -- its measured
    clean per-task means as latencies, the lanes' J-preset injection table and
    per-edge comm delays -- with every task lasting max(nominal + pad, nominal
    * X), the K11 rule (rrfp_exec.cu lane_complete) with the same lognormal
    draws X (pipeline.lognormal_floor_tables).  Model vs measurement."""
    import paper_2605_18750_b200 as P
    from paper_2605_18750_b200.pipeline import lognormal_floor_tables
    from paper_2605_18750_b200.tables import DIR_IDX, key_of
    g = pipe.group
    w = g.w
    floors = lognormal_floor_tables(pipe.N, pipe.M, nominal, sigma, floor_seed, n_chunks=pipe.C)
    mw = (w.num_microbatches + 31) // 32
    inj = {}
    for t, lat in w.latency.items():
        pad = g.injected.get(t, 0)
        fl = floors[t.stage][DIR_IDX[t.direction], key_of(t.microbatch, t.chunk, mw)] if sigma > 0 else 0.0
        inj[t] = int(max(lat + pad, fl) - lat)
    if name == "1f1b":
        _, m = P.run_fixed(P.build_1f1b_schedule(w), w, injected_delays=inj, record_trace=False)
    else:
        from paper_2605_18750_b200.engine import build_trace_metrics, replay_tables
        from paper_2605_18750_b200.tables import lower
        tb = lower(w, g.hint, g.tables.desc.buffer_limit, g._seed, None, g._tp, injected=inj)
        ev, res = replay_tables(tb)
        _, m = build_trace_metrics(w, ev, res, record_trace=False)
    return round(m.makespan / 1e3, 2)


def emulated_pp(args, cfg):
    """PP=N on ONE B200 (--emulate-pp N): N device lanes in this process, each
    stage on its own disjoint SM partition (CUDA green context, 16 SMs at N=8):
    every kernel of a stage's bodies -- GEMMs, attention, LayerNorm -- runs only
    on its partition, so an idle stage's SMs stay idle as on separate GPUs.
    Mailboxes in local memory.  Same kernels, dispatcher and injected jitter as
    the multi-GPU run; 1F1B vs BF vs BFW at every --sigmas value.  (--no-green:
    only the GEMM grids are capped and idle SMs are borrowed by other stages.)"""
    import gc
    import math
    import torch
    from paper_2605_18750_b200.jitter import PRESETS, JitterConfig
    from paper_2605_18750_b200.pipeline import GpuPipeline
    from paper_2605_18750_b200.runtime import dispatch_latency
    from paper_2605_18750_b200.workload import CommDelay
    N = args.emulate_pp
    cap = (torch.cuda.get_device_properties(0).multi_processor_count // N) & ~1
    combos = jitter_combos(args)
    # a stage on 148/N SMs runs ~N x slower than on its own GPU: the absolute-us
    # parts of the jitter (J-preset base delay, jitter.py:55-60; the lognormal
    # comm-delay median) are stretched by the same factor so the emulated pads
    # relate to the task times as they would on N GPUs (1 = unscaled)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    jscale = args.emu_jitter_scale if args.emu_jitter_scale > 0 else n_sm / cap

    def preset(jname):
        j = PRESETS[jname]
        return JitterConfig(j.probability, int(round(j.base_delay * jscale)), j.scale, j.level)
    out = {"n_stages": N, "gemm_sm_cap": cap, "green_partitions": bool(args.green),
           "definition": emulated_pp.__doc__.split("\n\n")[0].replace("\n", " ").replace("    ", " "),
           "jitter_time_scale": round(jscale, 3), "variants": {}}
    cur = torch.cuda.current_stream()
    for name, hint, mode in (("1f1b", "bf", "fixed"), ("bf", "bf", "free"), ("bfw", "bfw", "free")):
        t0 = time.perf_counter()
        # (built without jitter: the nominal task times below must be clean)
        pipe = GpuPipeline(cfg, N, args.mb, hint=hint, mode=mode, jitter=PRESETS["J0"],
                           head_cost=args.head_cost, gemm_sm_cap=cap, w_split=args.w_split,
                           green=args.green, split=stage_split(args))
        out["gemm_sm_cap"] = getattr(pipe, "green_sms", cap) if args.green else cap
        build_s = time.perf_counter() - t0
        for _ in range(2):
            pipe.step()
        nominal = pipe.nominal_us()
        pipe.set_nominal_latency(nominal)      # J-preset pads scale with the measured task times
        for jname, sigma in combos:
            pipe.group.set_jitter(preset(jname))
            comm = CommDelay()
            if sigma > 0:
                cu = args.comm_us * jscale
                comm = CommDelay(kind="lognormal", mu=math.log(cu), sigma=sigma, lo=0,
                                 hi=int(cu * 50), seed=17)
            pipe.group.set_comm_delay(comm)
            pipe.set_lognormal_jitter(sigma, seed=11, nominal_us=nominal)
            pipe.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(torch.cuda.current_device()) as clk:
                e0.record(cur)
                for _ in range(args.steps):
                    pipe.launch()
                    pipe.wait()
                for st in pipe.group.streams.values():
                    cur.wait_stream(st)
                e1.record(cur)
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            tr, met = pipe.trace()
            if args.trace_dir:
                os.makedirs(args.trace_dir, exist_ok=True)
                tr.dump_jsonl(os.path.join(args.trace_dir, f"pp{N}_{name}_sigma{sigma}.jsonl"))
            out["variants"][f"{name}@{jname}+sigma{sigma}"] = {
                "iter_s": round(1000.0 / ms, 4), "ms": round(ms, 2),
                "bubble_fraction": round(met.bubble_fraction(), 4), "build_s": round(build_s, 1),
                "dispatch": dispatch_latency(tr, N),
                # all N stages share this GPU's power budget: a schedule that keeps
                # more stages busy runs at a lower SM clock than on N separate GPUs
                "sm_mhz": clk.summary()["sm_mhz"]}
            try:
                pred = replay_prediction(pipe, name, sigma, nominal)
                out["variants"][f"{name}@{jname}+sigma{sigma}"]["model_ms"] = pred
                out["variants"][f"{name}@{jname}+sigma{sigma}"]["model_err"] = round(ms / pred - 1.0, 4)
            except Exception as exc:      # a model failure must not void the measurement
                _log(f"replay prediction failed: {exc!r}")
            _log(f"emulated PP={N} {name} {jname} sigma={sigma}: {ms:.1f} ms")
        pipe.close()
        del pipe
        gc.collect()
        torch.cuda.empty_cache()
    v = out["variants"]
    for jname, sigma in combos:
        base = v.get(f"1f1b@{jname}+sigma{sigma}")
        for name in ("bf", "bfw"):
            x = v.get(f"{name}@{jname}+sigma{sigma}")
            if base and x:
                x["speedup_vs_1f1b"] = round(base["ms"] / x["ms"], 4)
                if base.get("sm_mhz") and x.get("sm_mhz"):
                    # the stages share one power-capped GPU here: the speed-up in SM cycles
                    # (ms x median SM clock), what separate GPUs would see at equal clocks
                    x["speedup_vs_1f1b_equal_clock"] = round(
                        base["ms"] * base["sm_mhz"] / (x["ms"] * x["sm_mhz"]), 4)
    return out


def gather_trace(pipe, dist, world):
    """Wall trace + metrics of the last iteration over every rank's device events."""
    from paper_2605_18750_b200 import _lib
    from paper_2605_18750_b200.runtime import wall_trace
    ev, t0n = pipe.last_events
    if dist:
        allev = [None] * world
        dist.all_gather_object(allev, pipe.aligned_events())   # one clock: rank 0's
        ev = []
        for lst, _ in allev:
            for t in lst:
                x = _lib.Event()
                x.t0, x.t1, x.kind, x.stage, x.rank, x.task = t
                ev.append(x)
        t0n = min(t for _, t in allev)
    return wall_trace(pipe.workload, ev, t0n)


def timed_steps(pipe, steps, dist, barrier):
    """K iterations between CUDA events on the lane stream; max over ranks (ms/step)."""
    import torch
    lane_stream = pipe.group.streams[next(iter(pipe.group.streams))]
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(lane_stream)
    for _ in range(steps):
        pipe.launch()
        pipe.wait()
    e1.record(lane_stream)
    barrier()
    ms = e0.elapsed_time(e1) / steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    return ms


def jitter_combos(args):
    """(J-preset, sigma) operating points of the comparison runs: the first
    --compare-jitter preset at every --sigmas value (0 always included), each
    further preset at the largest sigma (default: J0 x {0, 0.5} + J2, J3 x 0.5,
    the regime SURVEY 6.3 puts the >= 1.5x target in)."""
    js = [j for j in args.compare_jitter.split(",") if j]
    sigmas = sorted({0.0, *[float(x) for x in args.sigmas.split(",") if x]})
    out = [(js[0], sg) for sg in sigmas]
    out += [(j, sigmas[-1]) for j in js[1:]]
    return out


def compare_variants(cfg, args, world, dist, barrier):
    """Same kernels, same box: fixed-order 1F1B vs RRFP (BF, BFW) under the
    J-preset jitter table (--compare-jitter) and injected lognormal compute +
    comm jitter for every sigma of --sigmas (config 5's sweep; draws keyed by
    task / edge, so every variant sees identical perturbations).  One build per
    variant; per sigma: new floor + comm tables, one warm step, K device-timed
    steps.  Nominal task times = the variant's own clean (sigma 0) iteration."""
    import gc
    import math
    import torch
    from paper_2605_18750_b200.jitter import PRESETS
    from paper_2605_18750_b200.workload import CommDelay
    out = {}
    combos = jitter_combos(args)
    jit = PRESETS["J0"]     # nominal task times are measured without injected jitter
    for name, hint, mode in (("1f1b", "bf", "fixed"), ("bf", "bf", "free"), ("bfw", "bfw", "free")):
        if name == "1f1b" and args.chunks > 1:
            continue          # 1F1B is undefined for interleaved chunks (baselines.py:72-75)
        if world == 1 and name == "bfw" and cfg.n_layer * args.mb > 8 * 32:
            continue          # PP=1 BFW keeps every W pending: memory-bound, meaningless
        pipe, stages = build_pipe(cfg, args, hint, mode, world, jit)
        if dist:
            pipe.calibrate_clocks()
        for _ in range(2):
            pipe.step()
        nominal = pipe.nominal_us()
        pipe.set_nominal_latency(nominal)      # J-preset pads scale with the measured task times
        for jname, sigma in combos:
            pipe.group.set_jitter(PRESETS[jname])
            comm = CommDelay()
            if sigma > 0:
                comm = CommDelay(kind="lognormal", mu=math.log(args.comm_us), sigma=sigma, lo=0,
                                 hi=int(args.comm_us * 50), seed=17)
            pipe.group.set_comm_delay(comm)
            pipe.set_lognormal_jitter(sigma, seed=11, nominal_us=nominal)
            pipe.step()
            ms = timed_steps(pipe, args.steps, dist, barrier)
            tr, met = gather_trace(pipe, dist, world)
            key = f"{name}@{jname}+sigma{sigma}"
            out[key] = {"iter_s": round(1000.0 / ms, 4), "ms": round(ms, 2),
                        "tokens_per_s": round(1000.0 / ms * args.mb * cfg.seq, 1),
                        "bubble_fraction": round(met.bubble_fraction(), 4)}
            if not dist or dist.get_rank() == 0:   # (rank 0 holds the gathered trace)
                from paper_2605_18750_b200.runtime import dispatch_latency
                out[key]["dispatch"] = dispatch_latency(tr, pipe.workload.num_stages)
            _log(f"variant {name} {jname} sigma={sigma}: {ms:.1f} ms")
        pipe.close()
        del pipe, stages
        gc.collect()
        torch.cuda.empty_cache()
    for jname, sigma in combos:
        base = out.get(f"1f1b@{jname}+sigma{sigma}")
        if base:
            for name in ("bf", "bfw"):
                v = out.get(f"{name}@{jname}+sigma{sigma}")
                if v:
                    v["speedup_vs_1f1b"] = round(base["ms"] / v["ms"], 4)
    return out


def p2p_block(pipe, cfg, args, dist, world, clock_cal):
    """NVLink evidence of the N>1 run (rank 0 reports, every rank measures):
    the mailbox store of one [S, D] bf16 activation (8 MiB at 1.3B) into the
    NEXT stage's slot on the peer GPU vs into a local buffer (our copy kernel,
    CUDA events, 20 reps), the FC2 GEMM with its epilogue writing the peer
    mailbox vs a local output (the fused K1 path), the device flag round trip
    (clock ping-pong), and the TP all-reduce (R-1 peer partials per call)."""
    import ctypes as C
    import torch
    from paper_2605_18750_b200 import _lib
    from paper_2605_18750_b200 import kernels as K
    L = _lib.lib()
    S, D, Fd = cfg.seq, cfg.d_model, cfg.d_ff
    st = pipe.vstages[0]
    out = {"rank": dist.get_rank()}
    stream = torch.cuda.current_stream()
    try:
        _p2p_measure(out, pipe, st, L, K, S, D, Fd, stream, dist, clock_cal)
    except Exception as e:       # a probe must never cost the run (or hang the gather)
        out["error"] = repr(e)[:200]
    allv = [None] * world
    dist.all_gather_object(allv, out)
    return allv


def _p2p_measure(out, pipe, st, L, K, S, D, Fd, stream, dist, clock_cal):
    import ctypes as C
    import torch
    from paper_2605_18750_b200 import _lib

    def timeit(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e-3

    if st.fwd_out is not None:
        peer = st.fwd_out[0][0]
        src = torch.randn(S, D, device="cuda").to(torch.bfloat16)
        local = torch.empty_like(src)
        nbytes = S * D * 2

        def cp(dst):
            return lambda: _lib.check(L.rrfp_copy_rows(C.c_void_p(dst.data_ptr()), C.c_longlong(D * 2),
                                                       C.c_void_p(src.data_ptr()), C.c_longlong(D * 2), S,
                                                       C.c_longlong(D * 2), C.c_void_p(stream.cuda_stream)))
        tp_, tl = timeit(cp(peer)), timeit(cp(local))
        out["mailbox_copy"] = {"bytes": nbytes, "peer_gbs": round(nbytes / tp_ / 1e9, 1),
                               "local_gbs": round(nbytes / tl / 1e9, 1), "peer_us": round(tp_ * 1e6, 1)}
        act = torch.randn(S, Fd, device="cuda").to(torch.bfloat16)
        w2 = torch.randn(D, Fd, device="cuda").to(torch.bfloat16)
        bias = torch.zeros(D, device="cuda").to(torch.bfloat16)
        gp = timeit(lambda: K.gemm(act, w2, peer, epi=K.EPI_RESID, bias=bias, r=src), 10)
        gl = timeit(lambda: K.gemm(act, w2, local, epi=K.EPI_RESID, bias=bias, r=src), 10)
        out["fc2_epilogue_to_mailbox"] = {"peer_us": round(gp * 1e6, 1), "local_us": round(gl * 1e6, 1),
                                          "tflops_peer": round(2 * S * D * Fd / gp / 1e12, 1)}
    if clock_cal:
        out["flag_round_trip_ns_best"] = clock_cal["best_rtt_ns"]
    comm = getattr(pipe, "comm", None)
    if comm is not None:
        dst = torch.empty(S, D, device="cuda").to(torch.bfloat16)
        dist.barrier()
        t = timeit(lambda: comm.allreduce([dst]), 20)
        moved = (comm.size - 1) * S * D * 2
        out["tp_allreduce"] = {"us": round(t * 1e6, 1), "peer_read_gbs": round(moved / t / 1e9, 1),
                               "bytes_peer_per_call": moved}


def scheduler_baseline(task_us, n_meas, args, device="cuda"):
    """SURVEY 8d CPU item (i): the reference's virtual-clock schedulers
    (engine.run_rrfp, baselines.run_fixed -- the oracle's restatement, one
    core) vs the device replay kernel on IDENTICAL tables built from this
    run's measured per-task times, PP 4/8 x M 16/32; microseconds per task."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rrfp_oracle as O
    import paper_2605_18750_b200 as P
    f_tot = sum(task_us["F"])
    b_tot = sum(task_us["B"])
    out = []
    for n in (4, 8):
        for m in (16, 32):
            lat = {}
            for s_ in range(n):
                for mb in range(m):
                    lat[P.TaskId(s_, mb, 0, "F")] = max(1, int(f_tot / n))
                    lat[P.TaskId(s_, mb, 0, "B")] = max(1, int(b_tot / n))
            w = P.Workload(num_stages=n, num_microbatches=m, num_chunks=1, tp_group_size=1, latency=lat)
            ow = O.from_workload_json(w.to_json())
            tasks = w.task_count()
            row = {"pp": n, "mb": m, "tasks": tasks}
            for name, fn in (("run_rrfp_cpu", lambda: O.run_rrfp(ow, "bf", 32, 0, "J3")),
                             ("run_fixed_cpu", lambda: O.run_fixed(O.one_f_one_b(ow), ow)),
                             ("replay_kernel_gpu", lambda: P.run_rrfp(w, "bf", 32, 0,
                                                                      jitter=P.JITTER_PRESETS["J3"],
                                                                      device=device))):
                fn()
                k, t0 = 0, time.perf_counter()
                while time.perf_counter() - t0 < 0.5 or k < 2:
                    fn()
                    k += 1
                row[name + "_us_per_task"] = round((time.perf_counter() - t0) / k / tasks * 1e6, 2)
            out.append(row)
    return {"definition": scheduler_baseline.__doc__.split("\n\n")[0].strip().replace("\n", " "),
            "note": "replay_kernel_gpu includes the table upload and the event read-back per call",
            "rows": out}


def cpu_baseline(args, n, task_us):
    """oracle.run_live (the reference's threaded CPU runtime, restated) driving the
    same task graph with this run's measured per-task times; ~10 s sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import rrfp_oracle as O
    dec = args.hint == "bfw"
    lat = {}
    for s_ in range(n):
        for mb in range(args.mb):
            lat[("F", s_, mb, 0)] = max(1, int(task_us["F"][s_]))
            lat[("B", s_, mb, 0)] = max(1, int(task_us["B"][s_]))
            if dec:
                lat[("W", s_, mb, 0)] = max(1, int(task_us["W"][s_]))
    w = {"N": n, "M": args.mb, "C": 1, "R": 1, "lat": lat, "comm": {"kind": "constant", "value": 0},
         "dec": dec, "beta": 0.5}
    hint = "bf" if args.hint == "1f1b" else args.hint
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 10.0 or k < 1:
        O.run_live(w, hint, 32, 1.0, seed=0)
        k += 1
    dt = (time.perf_counter() - t0) / k
    out = {"value": round(1.0 / dt, 4), "unit": "iter/s", "cores": 3 * n, "kind": "port",
           "os_cpu_count": os.cpu_count(), "sched_affinity": len(os.sched_getaffinity(0)),
           "sample": f"{k} iterations of oracle.run_live ({3 * n} threads, GIL-bound) on this run's "
                     f"measured per-task times, PP={n}, M={args.mb}"}
    try:
        out["scheduler"] = scheduler_baseline(task_us, n, args)
    except Exception as e:     # never cost the measurement
        out["scheduler"] = {"error": repr(e)[:200]}
    return out


def reexec_torchrun(n):
    """``python bench.py --gpus N`` (no torchrun): one process per GPU, launched
    the way the driver launches the N > 1 runs; returns the exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    _log(f"re-exec under torchrun: {n} ranks")
    return subprocess.run(cmd).returncode


def dry_run(args):
    """The launch plan every rank resolved (rendezvous over gloo when N > 1)."""
    rank, world, local = dist_env()
    plan = {"n_gpus": world, "pp": world // args.tp if world > 1 else 1, "tp": args.tp,
            "chunks": args.chunks, "impl": args.impl, "rank_to_stage":
            [[r // args.tp, r % args.tp] for r in range(world)], "dry_run": True}
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        allp = [None] * world
        dist.all_gather_object(allp, {"rank": rank, "local_rank": local})
        plan["ranks"] = allp
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(plan), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--hint", default="bf", choices=["bf", "bfw", "fb", "bprio", "fprio", "1f1b"])
    ap.add_argument("--mb", type=int, default=32)
    ap.add_argument("--layers", type=int, default=None, help="default: 24 (1.3b) / 32 (7b)")
    ap.add_argument("--model", default="1.3b", choices=["1.3b", "7b", "mm"],
                    help="1.3b (config 2), 7b (config 3 with --tp 2), mm = ViT-H + 7B (config 4)")
    ap.add_argument("--tp", type=int, default=1, help="tensor-parallel group size per stage (config 3: 2)")
    ap.add_argument("--chunks", type=int, default=1, help="interleaved virtual stages per GPU (C)")
    ap.add_argument("--head-cost", dest="head_cost", type=float, default=1.4,
                    help="LM head + loss of the last stage in layer-equivalents for the balanced layer "
                         "split (measured: F 400 + B 650 us vs 762 us per layer); 0 = even split")
    ap.add_argument("--jitter", default="J0")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--compare", dest="compare", action="store_true", default=None,
                    help="also time fixed 1F1B / BF / BFW (default on for N>1)")
    ap.add_argument("--no-compare", dest="compare", action="store_false")
    ap.add_argument("--sigmas", default="0.5",
                    help="comma list of lognormal compute+comm jitter sigmas of the comparison runs "
                         "(config 5 sweep: 0,0.1,0.2,0.3,0.4,0.5); sigma 0 is always included")
    ap.add_argument("--emu-jitter-scale", dest="emu_jitter_scale", type=float, default=0.0,
                    help="emulated PP: stretch the J-preset base delay and the comm-delay median by this "
                         "factor (0 = auto: SMs of the GPU / SMs of a stage partition)")
    ap.add_argument("--compare-jitter", dest="compare_jitter", default="J0,J2,J3",
                    help="comma list of J-preset jitter tables (jitter.py PRESETS) for the comparison runs: "
                         "the first at every --sigmas value, the others at the largest sigma")
    ap.add_argument("--comm-us", dest="comm_us", type=float, default=100.0)
    ap.add_argument("--w-split", dest="w_split", default="fc", choices=["fc", "all"],
                    help="BFW: weight gradients deferred to the W task (fc: FC1/FC2; all: all four)")
    ap.add_argument("--split", default="half", choices=["half", "layer"],
                    help="GPT stage boundaries: at half-layers (attention | MLP, balanced; default) or layers")
    ap.add_argument("--no-green", dest="green", action="store_false",
                    help="emulation without SM partitions (GEMM grids capped only)")
    ap.add_argument("--trace-dir", dest="trace_dir", default=None,
                    help="write each emulated variant's wall trace (JSONL) here")
    ap.add_argument("--emulate-only", dest="emulate_only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--emulate-pp", dest="emulate_pp", type=int, default=8,
                    help="(1 GPU) also run an emulated PP=N pipeline: N lanes, GEMMs on 148/N SMs each, "
                         "1F1B vs BF vs BFW at every --sigmas (default 8; 0 = off)")
    ap.add_argument("--emulate-pp-extra", dest="emulate_pp_extra", default="2,4",
                    help="(1 GPU) further emulated pipeline depths, J0 jitter only (default 2,4; '' = none)")
    ap.add_argument("--dry-run", dest="dry_run", action="store_true",
                    help="resolve the launch (re-exec under torchrun for --gpus N > 1, rendezvous) and "
                         "print the plan; no CUDA")
    args = ap.parse_args()
    rank, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.emulate_only and \
            (args.impl == "ours" or args.dry_run):
        sys.exit(reexec_torchrun(args.gpus))
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; one process per GPU "
                         f"(torchrun --nproc-per-node {args.gpus})")
    if args.dry_run:
        return dry_run(args)
    if args.emulate_only:
        import torch
        torch.cuda.set_device(0)
        print(json.dumps(emulated_pp(args, model_config(args))), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
