"""bench.py's JSON contract on CPU: the reference arm (the reference's CPU
runtime on the host cores) and the virtual-clock pipeline model (host twin)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--mb", "4"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["layer_split"] == [24]


def test_pipeline_model_on_host_twin():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2605_18750_b200.model import GPTConfig
    args = argparse.Namespace(head_cost=1.4, mb=8, comm_us=100.0, model="1.3b", split="layer")
    out = bench.pipeline_model(args, GPTConfig(), {"F": [6400.0], "B": [12700.0]}, 1, pps=(2, 8),
                               device="cpu")
    assert out["pp8"]["layers"] == [4, 3, 3, 3, 3, 3, 3, 2]
    args.split = "half"
    half = bench.pipeline_model(args, GPTConfig(), {"F": [6400.0], "B": [12700.0]}, 1, pps=(8,),
                                device="cpu")
    assert half["pp8"]["layers"] == [3.42, 3.58, 3, 3, 3, 3, 3, 2.0]   # heavier stages first
    # without jitter the bottleneck sets the pace: the balanced split is faster
    assert half["pp8"]["sigma0.0"]["1f1b"]["ms"] <= out["pp8"]["sigma0.0"]["1f1b"]["ms"]
    assert half["pp8"]["sigma0.0"]["bfw"]["ms"] < out["pp8"]["sigma0.0"]["bfw"]["ms"]
    for pp in ("pp2", "pp8"):
        for sig in ("sigma0.0", "sigma0.5"):
            r = out[pp][sig]
            assert r["1f1b"]["ms"] > 0 and r["bf"]["speedup_vs_1f1b"] > 0.8
    # jitter makes every schedule slower
    assert out["pp8"]["sigma0.5"]["1f1b"]["ms"] > out["pp8"]["sigma0.0"]["1f1b"]["ms"]
    # the (sigma x J-preset) operating grid at PP=8
    g = half["pp8_grid"]
    assert g["levels"] == ["J0", "J1", "J2", "J3"] and len(g["sigmas"]) == 6
    for key in ("bfw_speedup", "bf_speedup", "bubble_1f1b", "bubble_bfw"):
        assert all(len(g[key][j]) == 6 for j in g["levels"])
    assert all(v > 0.9 for j in g["levels"] for v in g["bfw_speedup"][j])
    assert all(g["bubble_bfw"][j][i] <= g["bubble_1f1b"][j][i] + 0.02 for j in g["levels"] for i in range(6))
    assert all(g["bfw_speedup"][j][i] >= 1.5 for j, s in g["points_bfw_ge_1p5"]
               for i in [g["sigmas"].index(s)])


def test_dispatch_latency_from_trace():
    """Back-to-back gaps count only when the next task was ready at the previous
    one's end; otherwise the arrival -> start delay is reported."""
    from paper_2605_18750_b200.runtime import dispatch_latency
    from paper_2605_18750_b200.trace import Trace, TraceEvent
    ev = [TraceEvent(0, 100, 0, None, 0, 0, "F", "exec"),
          TraceEvent(120, 220, 0, None, 1, 0, "F", "exec"),      # stage-0 F: ready -> gap 20
          TraceEvent(150, 150, 1, 0, 0, 0, "F", "recv"),         # (recvs carry rank 0, TP=1 execs None)
          TraceEvent(100, 260, 1, None, 0, 0, "F", "exec"),      # (first on its lane)
          TraceEvent(300, 300, 1, 0, 1, 0, "F", "recv"),
          TraceEvent(310, 400, 1, None, 1, 0, "F", "exec"),      # arrived after the end: react 10
          TraceEvent(425, 600, 1, None, 0, 0, "B", "exec"),      # last stage B after its F: gap 25
          TraceEvent(240, 300, 0, None, 0, 0, "F", "send")]
    tr = Trace(events=ev) if "events" in Trace.__dataclass_fields__ else Trace(ev)
    d = dispatch_latency(tr, 2)
    assert d["back_to_back_gap_us"]["n"] == 2 and d["back_to_back_gap_us"]["p50"] == 25
    assert d["arrival_to_start_us"] == {"p50": 10, "p90": 10, "n": 1}


def _json_line(p):
    return json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])


def test_gpus_n_is_self_sufficient_on_cpu():
    """`python bench.py --gpus 2` without torchrun: our arm re-executes itself
    under torch.distributed.run with 2 ranks (dry run: rendezvous + plan, no
    CUDA) and the reference arm runs PP=2 on rank 0."""
    env = dict(os.environ, RRFP_SAME_DEVICE="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    plan = _json_line(p)
    assert plan["n_gpus"] == 2 and plan["pp"] == 2 and len(plan["ranks"]) == 2
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--mb", "4"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    line = _json_line(p)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "pp2"
    assert line["cpu_baseline"]["os_cpu_count"] >= 1


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr


def test_reference_arm_refuses_1f1b():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--hint", "1f1b",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "unavailable" in _json_line(p)


def test_jitter_combos_default_includes_j3():
    sys.path.insert(0, ROOT)
    import bench
    args = argparse.Namespace(compare_jitter="J0,J3", sigmas="0.5")
    assert bench.jitter_combos(args) == [("J0", 0.0), ("J0", 0.5), ("J3", 0.5)]
