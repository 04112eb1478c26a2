"""Dispatcher cost per decision on the device lanes ("report ns per
decision"): N lanes on one GPU, every task a 1 us spin body, so an iteration is
almost all dispatch.  Reports back-to-back gap and arrival->start percentiles
(runtime.dispatch_latency) and makespan / task."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_18750_b200 as P
from paper_2605_18750_b200.runtime import dispatch_latency, run_gpu
from paper_2605_18750_b200.workload import constant

out = {}
for N, M, hint in [(1, 32, "bf"), (4, 32, "bf"), (8, 32, "bf"), (8, 32, "bfw")]:
    spec = P.GeneratorSpec(num_stages=N, num_microbatches=M, forward=constant(2),
                           backward=constant(2), decompose_backward=hint == "bfw")
    w = P.generate_workload(spec, 0)
    res = []
    for it in range(4):
        tr, met = run_gpu(w, hint, 32, seed=0)
        res.append((met.makespan, dispatch_latency(tr, N)))
    mk, d = res[-1]
    out[f"pp{N}_{hint}"] = {"makespan_us": mk, "tasks_per_lane": w.task_count() // N,
                            "us_per_task_critical_lane": round(mk / (w.task_count() // N), 2), **d}
    print(f"pp{N} {hint}", json.dumps(out[f"pp{N}_{hint}"]), flush=True)
print(json.dumps(out))
