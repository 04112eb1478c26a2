"""Pin the CPU oracle (oracle/rrfp_oracle.py) against the real reference's outputs."""
import pytest

import rrfp_oracle as O
from golden_util import engine_cases, load

CASES = engine_cases()


def _workload(case):
    return O.generate(case["spec"], case["seed"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_generator_matches_reference(case):
    w = _workload(case)
    ref = O.from_workload_json(case["workload"])
    assert w["lat"] == ref["lat"]
    assert w["comm"].get("seed", 0) == ref["comm"].get("seed", 0)


@pytest.mark.parametrize("case", [c for c in CASES if "deadlock" not in c],
                         ids=[c["name"] for c in CASES if "deadlock" not in c])
def test_tables_match_reference(case):
    w = _workload(case)
    inj = O.injection_table(w, case["jitter"], case["seed"])
    assert {O.task_key(t): v for t, v in inj.items()} == case["injection"]
    comm = {f"{O.task_key(s)}>{O.task_key(d)}": O.comm_delay_sample(w["comm"], s, d, k)
            for s, d, k in O.task_graph(w)}
    assert comm == case["comm_table"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_engine_matches_reference(case):
    w = _workload(case)
    tp = case.get("tp")
    if "deadlock" in case:
        with pytest.raises(O.DeadlockError):
            O.run_rrfp(w, case["hint"], case["limit"], case["seed"], case["jitter"], tp,
                       ranked=[tuple(e) for e in case.get("ranked") or ()])
        return
    ev, metrics = O.run_rrfp(w, case["hint"], case["limit"], case["seed"], case["jitter"], tp,
                             ranked=[tuple(e) for e in case.get("ranked") or ()])
    assert metrics == case["metrics"]
    for rank, per in case["exec"].items():
        got = O.exec_sequences(ev, w["N"], rank=int(rank))
        assert [[list(x) for x in s] for s in got] == per
    assert [list(e) for e in ev] == case["events"]


@pytest.mark.parametrize("case", [c for c in CASES if c.get("fixed") and "deadlock" not in c],
                         ids=[c["name"] for c in CASES if c.get("fixed") and "deadlock" not in c])
def test_fixed_1f1b_matches_reference(case):
    w = _workload(case)
    inj = O.injection_table(w, case["jitter"], case["seed"])
    ev, metrics = O.run_fixed(O.one_f_one_b(w), w, inj)
    got = O.exec_sequences(ev, w["N"])
    assert [[list(x) for x in s] for s in got] == case["fixed_exec"]
    assert metrics["makespan"] == case["fixed_metrics"]["makespan"]


APPENDIX_B = {  # SURVEY.md Appendix B golden table (1F1B / BF makespan + hash)
    ("J0", 0): (1183668, "ba37ada04651f3e9", 1044092, "d9f201da3671e6c4"),
    ("J0", 1): (1078483, "55e265051888f032", 949039, "58d8a5d7b78a3f8f"),
    ("J0", 2): (1239962, "52fedcf539bb8a6b", 1097864, "4eb1f0a7e2642c46"),
    ("J3", 0): (1831012, "d193d53fa58a2c40", 1516807, "4721691a1dda1034"),
    ("J3", 1): (1742388, "1ccbecb0182a4688", 1504689, "e71e498a918a0308"),
    ("J3", 2): (1910547, "0079f02974145562", 1606764, "a333b942a459a3e1"),
}


@pytest.mark.parametrize("level,seed", sorted(APPENDIX_B))
def test_appendix_b_hashes(level, seed):
    spec = {"num_stages": 4, "num_microbatches": 16,
            "forward": {"kind": "lognormal", "mu": 10.0, "sigma": 0.35, "lo": 8000, "hi": 60000},
            "backward": {"kind": "lognormal", "mu": 10.2, "sigma": 0.35, "lo": 8000, "hi": 70000}}
    w = O.generate(spec, seed)
    inj = O.injection_table(w, level, seed)
    fev, fm = O.run_fixed(O.one_f_one_b(w), w, inj)
    bev, bm = O.run_rrfp(w, "bf", 32, seed, level)
    want = APPENDIX_B[(level, seed)]
    assert (fm["makespan"], O.dispatch_hash(fev, 4), bm["makespan"], O.dispatch_hash(bev, 4)) == want


def test_known_answers():
    kat = load("known_answers.json")
    for a, b, want in kat["ema"]:
        assert O.ema(a, b) == want
    # J3 formula from the reference's test_jitter.py:42-47 (gate 0.1, r 0.5, ema 10000)
    p, base, scale = O.JITTER["J3"]
    assert int(round(scale * max(base, 10000) * (0.5 + 0.5))) == 22500


def test_arbiter_snapshots():
    snaps = load("arbiter_snapshots.json")["snapshots"]
    assert len(snaps) > 1000
    for sn in snaps:
        v = O.View()
        v.fready = {tuple(x) for x in sn["fready"]}
        v.bready = {tuple(x) for x in sn["bready"]}
        v.admission = sn["admission"]
        v.wpend = {tuple(x) for x in sn["wpend"]}
        ctl = O.StageCtl(32, sn["C"], sn["M"])
        ctl.mode = {"normal": "normal", "drain_backward": "drain",
                    "focus_microbatch": "focus"}[sn["mode"]]
        ctl.focus = sn["focus"]
        ctl.phase = sn["phase"]
        ctl.done = {tuple(x) for x in sn["done"]}
        out = O.arbitrate(v, ctl, sn["hint"], sn["dec"], [tuple(e) for e in sn["ranked"]])
        want = (sn["out"][0], None if sn["out"][1] is None else tuple(sn["out"][1]))
        assert out == want, sn
