"""Generate the golden fixtures in tests/golden/ from the REAL reference.

TEST INFRASTRUCTURE.  Run in the build container only (needs
/root/reference, which does not exist on the GPU box):

    python oracle/gen_golden.py

The reference is read-only, so it is copied to /tmp and imported from
there.  Every fixture records the numpy version it was produced with
(the reference's RNG is numpy PCG64).
"""

from __future__ import annotations

import json
import os
import random
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg"
COPY = "/tmp/rrfp_ref_copy"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _import_reference():
    if not os.path.isdir(COPY):
        shutil.copytree(REF, COPY)
    sys.path.insert(0, os.path.join(COPY, "src"))
    import rrfp  # noqa: F401
    return rrfp


def corpus():
    """Deterministic list of engine cases covering the S1-S12 checklist."""
    cases = []
    # SURVEY App. B config 1 (BASELINE configs[0]): N=4, M=16 jitter-preset lognormals
    c1 = {"num_stages": 4, "num_microbatches": 16,
          "forward": {"kind": "lognormal", "mu": 10.0, "sigma": 0.35, "lo": 8000, "hi": 60000},
          "backward": {"kind": "lognormal", "mu": 10.2, "sigma": 0.35, "lo": 8000, "hi": 70000}}
    for level in ("J0", "J3"):
        for seed in (0, 1, 2):
            cases.append({"name": f"config1-{level}-s{seed}", "spec": c1, "seed": seed,
                          "hint": "bf", "limit": 32, "jitter": level, "tp": None,
                          "fixed": True})
    # the bundled configs (pkg/configs/*.json)
    cases.append({"name": "example", "spec": {
        "num_stages": 4, "num_microbatches": 8,
        "forward": {"kind": "uniform", "lo": 80, "hi": 120},
        "backward": {"kind": "uniform", "lo": 80, "hi": 120}},
        "seed": 1, "hint": "bf", "limit": 32, "jitter": "J0", "tp": None, "fixed": True})
    cases.append({"name": "heavy-multimodal", "spec": {
        "num_stages": 8, "num_microbatches": 24,
        "forward": {"kind": "uniform", "lo": 150, "hi": 250},
        "backward": {"kind": "uniform", "lo": 150, "hi": 250}, "heavy_prefix": 2.5},
        "seed": 3, "hint": "bf", "limit": 32, "jitter": "J0", "tp": None, "fixed": True})
    cases.append({"name": "interleaved-tp", "spec": {
        "num_stages": 4, "num_microbatches": 8, "num_chunks": 2, "tp_group_size": 2,
        "forward": {"kind": "lognormal", "mu": 4.8, "sigma": 0.4, "lo": 40, "hi": 400},
        "backward": {"kind": "lognormal", "mu": 5.0, "sigma": 0.4, "lo": 40, "hi": 500},
        "comm_delay": {"kind": "uniform", "lo": 5, "hi": 30, "seed": 7}},
        "seed": 7, "hint": "bf", "limit": 8, "jitter": "J1",
        "tp": {"cost": 5, "skew_lo": 0, "skew_hi": 20}, "fixed": False})
    # randomized sweep over hints / chunks / ranks / limits / comm / jitter
    rng = random.Random(2605)
    hints = ["bf", "fb", "bprio", "fprio", "bfw", "external"]
    for i in range(48):
        n = rng.choice([1, 2, 3, 4, 8])
        m = rng.choice([1, 2, 3, 5, 8, 16])
        c = rng.choice([1, 1, 2, 3])
        r = rng.choice([1, 1, 1, 2, 4])
        hint = hints[i % len(hints)]
        dec = hint == "bfw" or (hint == "external" and rng.random() < 0.5)
        fd = rng.choice([{"kind": "uniform", "lo": 1, "hi": 300},
                         {"kind": "lognormal", "mu": 5.0, "sigma": 0.5, "lo": 20, "hi": 900},
                         {"kind": "constant", "value": 100}])
        bd = rng.choice([{"kind": "uniform", "lo": 1, "hi": 400},
                         {"kind": "lognormal", "mu": 5.3, "sigma": 0.5, "lo": 20, "hi": 900},
                         {"kind": "constant", "value": 100}])
        comm = rng.choice([{"kind": "constant", "value": 0}, {"kind": "constant", "value": 7},
                           {"kind": "uniform", "lo": 0, "hi": 40},
                           {"kind": "lognormal", "mu": 2.5, "sigma": 0.6, "lo": 0, "hi": 80}])
        spec = {"num_stages": n, "num_microbatches": m, "num_chunks": c, "tp_group_size": r,
                "forward": fd, "backward": bd, "comm_delay": comm, "decompose_backward": dec,
                "heavy_last": rng.choice([1.0, 1.0, 1.7]),
                "heavy_prefix": rng.choice([1.0, 1.0, 2.5])}
        ranked = None
        if hint == "external":
            opts = [["F", "asc"], ["F", "desc"], ["B", "asc"], ["B", "desc"], ["W", "asc"]]
            rng.shuffle(opts)
            ranked = opts[:rng.randint(1, 4)]
        tp = None
        if r > 1:
            tp = {"cost": rng.choice([0, 5, 11]), "skew_lo": 0, "skew_hi": rng.choice([0, 25, 60])}
        cases.append({"name": f"rand{i:02d}", "spec": spec, "seed": rng.randint(0, 999),
                      "hint": hint, "ranked": ranked, "limit": rng.choice([1, 2, 4, 32]),
                      "jitter": rng.choice(["J0", "J1", "J3"]), "tp": tp,
                      "fixed": c == 1 and not dec})
    # wide ready sets (more than 32 microbatches: multi-word bitmasks on the device),
    # limits below M (backpressure), and the config-2/5 shape (PP=8, M=32, BFW)
    logn = lambda mu, hi: {"kind": "lognormal", "mu": mu, "sigma": 0.4, "lo": 20, "hi": hi}
    wide = [
        ("wide-m40", {"num_stages": 4, "num_microbatches": 40, "forward": logn(5.0, 900),
                      "backward": logn(5.3, 900)}, "bf", None, 32, "J1", None, True),
        ("wide-m64-c2-bfw", {"num_stages": 4, "num_microbatches": 64, "num_chunks": 2,
                             "decompose_backward": True, "forward": logn(5.0, 900),
                             "backward": logn(5.3, 900),
                             "comm_delay": {"kind": "uniform", "lo": 0, "hi": 40, "seed": 3}},
         "bfw", None, 16, "J3", None, False),
        ("pp8-m32-bfw", {"num_stages": 8, "num_microbatches": 32, "decompose_backward": True,
                         "forward": logn(6.0, 2000), "backward": logn(6.6, 4000),
                         "comm_delay": {"kind": "lognormal", "mu": 3.0, "sigma": 0.5, "lo": 0,
                                        "hi": 200, "seed": 17}},
         "bfw", None, 32, "J0", None, False),
        ("wide-m100-tp2", {"num_stages": 2, "num_microbatches": 100, "tp_group_size": 2,
                           "forward": logn(5.0, 900), "backward": logn(5.3, 900)},
         "fb", None, 32, "J1", {"cost": 5, "skew_lo": 0, "skew_hi": 25}, True),
        ("wide-m33-c3-external", {"num_stages": 3, "num_microbatches": 33, "num_chunks": 3,
                                  "forward": logn(5.0, 900), "backward": logn(5.3, 900)},
         "external", [["B", "asc"], ["F", "desc"]], 8, "J3", None, False),
    ]
    for name, spec, hint, ranked, limit, jit, tp, fixed in wide:
        cases.append({"name": name, "spec": spec, "seed": 11, "hint": hint, "ranked": ranked,
                      "limit": limit, "jitter": jit, "tp": tp, "fixed": fixed})
    return cases


def main():
    rrfp = _import_reference()
    from rrfp.arbitration import HintOrder, TpGroup
    from rrfp import engine as eng
    from rrfp.baselines import build_1f1b_schedule, run_fixed
    from rrfp.engine import run_rrfp
    from rrfp.jitter import PRESETS, build_injection_table
    from rrfp.workload import GeneratorSpec, build_task_graph, generate_workload

    os.makedirs(OUT, exist_ok=True)
    cases_out = []
    snapshots = []
    orig_arbitrate = eng.arbitrate

    for case in corpus():
        spec = GeneratorSpec.from_json(case["spec"])
        w = generate_workload(spec, case["seed"])
        hint = (HintOrder("external", tuple(tuple(e) for e in case["ranked"]))
                if case["hint"] == "external" else HintOrder(case["hint"]))
        jit = PRESETS[case["jitter"]]
        tp = None
        if case["tp"]:
            tp = TpGroup(group_size=w.tp_group_size, coordination_round_cost=case["tp"]["cost"],
                         skew_lo=case["tp"]["skew_lo"], skew_hi=case["tp"]["skew_hi"])
        taken = []

        def spy(buffers, hint_, bp, arb, workload, progress):
            d = orig_arbitrate(buffers, hint_, bp, arb, workload, progress)
            if len(taken) < 60:
                taken.append({
                    "fready": sorted([t.microbatch, t.chunk] for t in buffers.forward_ready),
                    "admission": None if buffers.admission is None else buffers.admission.microbatch,
                    "bready": sorted([t.microbatch, t.chunk] for t in buffers.backward_ready),
                    "wpend": sorted([t.microbatch, t.chunk] for t in buffers.weight_pending),
                    "mode": bp.mode, "focus": bp.focus_microbatch, "phase": arb.phase,
                    "done": sorted([mb, c, dd] for mb, c, dd in progress.done),
                    "hint": hint_.kind, "ranked": [list(e) for e in hint_.ranked],
                    "dec": workload.decompose_backward, "C": workload.num_chunks,
                    "M": workload.num_microbatches,
                    "out": [d.kind, None if d.task is None else [d.task.microbatch, d.task.chunk]],
                })
            return d

        eng.arbitrate = spy
        try:
            trace, metrics = run_rrfp(w, hint, case["limit"], case["seed"], jitter=jit, tp=tp)
        except eng.EngineDeadlockError as exc:
            out = dict(case)
            out.update({"workload": w.to_json(), "deadlock": str(exc)})
            cases_out.append(out)
            print("deadlock:", case["name"], exc)
            continue
        finally:
            eng.arbitrate = orig_arbitrate
        snapshots.extend(taken)
        r = w.tp_group_size
        seqs = {}
        for rank in range(r):
            per = [[] for _ in range(w.num_stages)]
            for e in trace.events:
                if e.event_kind == "exec" and (e.rank is None or e.rank == rank):
                    per[e.stage].append([e.direction, e.microbatch, e.chunk, e.t_start, e.t_end])
            seqs[str(rank)] = per
        coords = [[e.stage, e.t_start, e.t_end, e.direction, e.microbatch, e.chunk]
                  for e in trace.events if e.event_kind == "coord"]
        inj = build_injection_table(w, jit, case["seed"])
        comm = {f"{e.src.key()}>{e.dst.key()}": w.comm_delay.sample(e)
                for e in build_task_graph(w)}
        out = dict(case)
        out.update({
            "workload": w.to_json(),
            "injection": {t.key(): v for t, v in sorted(inj.items())},
            "comm_table": comm,
            "metrics": metrics.to_json(),
            "exec": seqs,
            "coord": coords,
            "events": [[e.t_start, e.t_end, e.stage, e.rank, e.microbatch, e.chunk,
                        e.direction, e.event_kind] for e in trace.events],
        })
        if case["fixed"]:
            ftrace, fmetrics = run_fixed(build_1f1b_schedule(w), w, injected_delays=inj)
            per = [[] for _ in range(w.num_stages)]
            for e in ftrace.events:
                if e.event_kind == "exec":
                    per[e.stage].append([e.direction, e.microbatch, e.chunk, e.t_start, e.t_end])
            out["fixed_exec"] = per
            out["fixed_metrics"] = fmetrics.to_json()
        cases_out.append(out)

    meta = {"numpy": np.__version__, "generator": "oracle/gen_golden.py",
            "reference": "/root/reference/pkg (rrfp 0.1.0)"}
    with open(os.path.join(OUT, "engine_cases.json"), "w") as f:
        json.dump({"meta": meta, "cases": cases_out}, f, separators=(",", ":"))
    with open(os.path.join(OUT, "arbiter_snapshots.json"), "w") as f:
        json.dump({"meta": meta, "snapshots": snapshots}, f, separators=(",", ":"))
    # unit known-answers from the reference's own tests (test_jitter.py:16-47)
    from rrfp.jitter import ema_update
    kat = {"meta": meta, "ema": [[10000, 20000, ema_update(10000, 20000)],
                                 [0, 0, ema_update(0, 0)], [5000, 5000, ema_update(5000, 5000)]]}
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(kat, f)
    print(f"{len(cases_out)} cases, {len(snapshots)} snapshots -> {os.path.abspath(OUT)}")


if __name__ == "__main__":
    main()
