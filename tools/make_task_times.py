"""Regenerate profiles/task_times_gpt1p3b.json (the per-stage F / B / B-input / W
task times bench.py --impl reference feeds the reference's CPU runtime) from a
PP=1 bench line: per-layer F and B from the measured per-microbatch task times
(LM head = 1.6 / 1.27 layer-equivalents of F / B, as bench.pipeline_model),
B-input / W as fractions of the fused B (bench.B_IN_FRAC / W_FRAC), stages split
as the bench splits them (model.split_units, half-layers, head cost 1.4).

    python tools/make_task_times.py profiles/r01_bench_pp1_r1end.json
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2605_18750_b200.model import ATTN_FRAC, split_units

src = sys.argv[1]
line = json.loads([l for l in open(src).read().splitlines() if l.startswith("{")][-1])
F, B = line["task_us"]["F"][0], line["task_us"]["B"][0]
L = 24
f_l, b_l = F / (L + 1.6), B / (L + 1.27)
w = {"full": 1.0, "attn": ATTN_FRAC, "mlp": 1.0 - ATTN_FRAC}
out = {"source": f"tools/make_task_times.py {os.path.relpath(src, ROOT)}: PP=1 GPT-1.3B M=32 task times "
                  f"F {F} us, B {B} us per microbatch (incl. LM head); per layer F {f_l:.1f}, B {b_l:.1f} us; "
                  f"B-input / W = {bench.B_IN_FRAC} / {bench.W_FRAC} of B (profiles/r01_task_times_ln_in_w.txt); "
                  "half-layer split with head cost 1.4; used by bench.py --impl reference",
       "unit": "us"}
for n in (1, 2, 4, 8):
    lay = [sum(w[p] for _, p in split_units(L, n, s, 1.4, "half" if n > 1 else "layer")) for s in range(n)]
    fs = [f_l * x + (1.6 * f_l if s == n - 1 else 0) for s, x in enumerate(lay)]
    bs = [b_l * x + (1.27 * b_l if s == n - 1 else 0) for s, x in enumerate(lay)]
    out[str(n)] = {"layers": [round(x, 2) for x in lay], "F": [round(x, 1) for x in fs],
                   "B": [round(x, 1) for x in bs], "Bin": [round(bench.B_IN_FRAC * x, 1) for x in bs],
                   "W": [round(bench.W_FRAC * x, 1) for x in bs]}
with open(os.path.join(ROOT, "profiles", "task_times_gpt1p3b.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out["8"]))
