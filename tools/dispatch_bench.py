"""Dispatcher cost per decision on the device lanes ("report ns per
decision"): N lanes on one GPU, every task a 1 us spin body, so an iteration is
almost all dispatch.  Reports back-to-back gap and arrival->start percentiles
(runtime.dispatch_latency) and makespan / task."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_18750_b200 as P
from paper_2605_18750_b200.runtime import LaneGroup, dispatch_latency, dispatcher_profile, run_gpu
from paper_2605_18750_b200.workload import constant

out = {}
for N, M, hint in [(1, 32, "bf"), (4, 32, "bf"), (8, 32, "bf"), (8, 32, "bfw")]:
    spec = P.GeneratorSpec(num_stages=N, num_microbatches=M, forward=constant(2),
                           backward=constant(2), decompose_backward=hint == "bfw")
    w = P.generate_workload(spec, 0)
    g = LaneGroup(w, hint, 32, 1.0, seed=0)
    try:
        for it in range(3):
            g.run_iteration(30.0)
        g.enable_profile(4096)
        events, t0s = g.run_iteration(30.0)
        tr, met = g.make_trace(events, t0s)
        prof = dispatcher_profile(g.profile(), body_us=2.0)
    finally:
        g.close()
    out[f"pp{N}_{hint}"] = {"makespan_us": met.makespan, "tasks_per_lane": w.task_count() // N,
                            "us_per_task_critical_lane": round(met.makespan / (w.task_count() // N), 2),
                            **dispatch_latency(tr, N), "step_kernel": prof}
    print(f"pp{N} {hint}", json.dumps(out[f"pp{N}_{hint}"]), flush=True)
print(json.dumps(out))
