"""Dev diagnostics on the box: small pipelines with tight watchdogs."""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("DIAG_DUMP", "50")), exit=True)
import torch
from paper_2605_18750_b200.model import GPTConfig
from paper_2605_18750_b200.pipeline import GpuPipeline

def run(name, cfg, n, m, hint, mode="free"):
    t = time.time()
    p = GpuPipeline(cfg, n, m, hint=hint, mode=mode)
    print(f"{name}: built in {time.time()-t:.1f}s", flush=True)
    for i in range(2):
        t1 = time.time()
        loss = p.step(watchdog_secs=15).item()
        tr, met = p.trace()
        ex = sorted(tr.execs(), key=lambda e: (e.stage, e.t_start))
        print(f"{name}: step {i} {time.time()-t1:.2f}s loss={loss:.4f} makespan={met.makespan}us "
              f"tasks={[(e.stage, e.direction, e.microbatch, e.t_end - e.t_start) for e in ex][:12]}", flush=True)
    p.close()

small = GPTConfig(n_layer=4, d_model=256, n_head=2, d_ff=1024, vocab=512, seq=256)
which = sys.argv[1]
cases = {
    "bf2": ("bf pp2 small", small, 2, 4, "bf"),
    "bf4": ("bf pp4 small", small, 4, 4, "bf"),
    "bfw1": ("bfw pp1 small", small, 1, 4, "bfw"),
    "L24M2": ("L24 M2", GPTConfig(), 1, 2, "bf"),
    "L4M8": ("L4 M8", GPTConfig(n_layer=4), 1, 8, "bf"),
}
run(*cases[which])
