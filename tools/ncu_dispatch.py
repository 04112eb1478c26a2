"""One device-dispatched iteration for an ncu capture of the dispatcher (dev tool):
PP=1 (or argv[1] lanes), M=8, 2 us spin bodies; the lane graph's WHILE node
relaunches lane_step_kernel once per decision."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_18750_b200 as P
from paper_2605_18750_b200.runtime import dispatch_latency, run_gpu
from paper_2605_18750_b200.workload import constant

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = P.generate_workload(P.GeneratorSpec(num_stages=N, num_microbatches=8, forward=constant(2),
                                        backward=constant(2)), 0)
tr, met = run_gpu(w, "bf", 32, seed=0)
print("makespan_us", met.makespan, dispatch_latency(tr, N), flush=True)
