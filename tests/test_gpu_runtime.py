"""Free-running device runtime (run_gpu) on the B200: live.run_live's test
strategy (pkg/tests/test_live.py), replay-mode bit-exactness of the lanes'
OWN decisions under the virtual clock, and a per-decision oracle check of
every arbitration the free-running lanes make."""
import pytest

import paper_2605_18750_b200 as P
from paper_2605_18750_b200.runtime import run_gpu
import rrfp_oracle as O

pytestmark = pytest.mark.gpu

SLACK = (5, 1.05, 400)   # wall traces: (lower_us, upper_rel, upper_abs_us)


def _tuples(trace):
    return [(e.t_start, e.t_end, e.stage, e.rank, e.microbatch, e.chunk, e.direction, e.event_kind)
            for e in trace.events]


def _oracle_w(w):
    return O.from_workload_json(w.to_json())


def _seqs(trace, n, rank=None):
    per = [[] for _ in range(n)]
    for e in sorted(trace.execs(), key=lambda e: e.t_start):
        if rank is None or e.rank in (None, rank):
            per[e.stage].append((e.direction, e.microbatch, e.chunk))
    return per


def _spec(n=4, m=8, **kw):
    return P.GeneratorSpec(num_stages=n, num_microbatches=m, forward=P.uniform(100, 300),
                           backward=P.uniform(150, 400), **kw)


def test_live_iteration_is_complete_and_valid():
    w = P.generate_workload(_spec(), 3)
    tr, m = run_gpu(w, "bf", 32, time_scale=1.0, seed=3)
    assert tr.clock == "wall"
    viol = O.validate(_tuples(tr), _oracle_w(w), slack=SLACK, clock="wall", scale=1.0)
    assert not viol, viol[:5]
    assert m.total_tasks == w.task_count()
    for s in m.per_stage:
        assert s.compute + s.blocking + s.tp_coord == m.makespan


def test_same_execution_multiset_as_virtual():
    w = P.generate_workload(_spec(3, 6), 1)
    tr, _ = run_gpu(w, "bf", 32, time_scale=1.0, seed=1)
    ev, _ = O.run_rrfp(_oracle_w(w), "bf", 32, 1)
    got = sorted((e.stage, e.direction, e.microbatch, e.chunk) for e in tr.execs())
    want = sorted((s, d, mb, c) for (_, _, s, r, mb, c, d, k) in ev if k == "exec")
    assert got == want


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_replay_mode_dispatch_bit_exact(seed):
    """North-star parity: under a replayed seeded readiness/jitter trace the
    device lanes execute exactly the oracle's per-stage dispatch order."""
    spec = P.GeneratorSpec(num_stages=4, num_microbatches=16,
                           forward=P.lognormal(10.0, 0.35, 8000, 60000),
                           backward=P.lognormal(10.2, 0.35, 8000, 70000))
    w = P.generate_workload(spec, seed)
    jit = P.JITTER_PRESETS["J3"]
    tr, _ = run_gpu(w, "bf", 32, time_scale=0.005, seed=seed, jitter=jit, mode="replay")
    ev, _ = O.run_rrfp(_oracle_w(w), "bf", 32, seed, "J3")
    want = [[(d, mb, c) for d, mb, c, _, _ in s] for s in O.exec_sequences(ev, 4)]
    assert _seqs(tr, 4) == want


def test_fixed_1f1b_follows_schedule():
    w = P.generate_workload(_spec(4, 8), 5)
    tr, m = run_gpu(w, "bf", 32, time_scale=1.0, seed=5, mode="fixed")
    sched = P.build_1f1b_schedule(w)
    want = [[(t.direction, t.microbatch, t.chunk) for t in st] for st in sched.per_stage_order]
    assert _seqs(tr, 4) == want
    viol = O.validate(_tuples(tr), _oracle_w(w), slack=SLACK, clock="wall", scale=1.0)
    assert not viol, viol[:5]


def test_tight_limits_never_stall():
    for limit in (1, 2):
        w = P.generate_workload(_spec(3, 6), 2)
        tr, m = run_gpu(w, "bf", limit, time_scale=1.0, seed=2, watchdog_secs=10)
        assert len(tr.execs()) == w.task_count()
        for s in range(3):
            lead = 0
            for e in sorted((e for e in tr.execs() if e.stage == s), key=lambda e: e.t_end):
                lead += 1 if e.direction == "F" else -1
                assert 0 <= lead <= limit


def test_weight_split_runs_all_w():
    w = P.generate_workload(_spec(3, 4, decompose_backward=True), 4)
    tr, m = run_gpu(w, "bfw", 32, time_scale=1.0, seed=4)
    assert sum(s.n_w for s in m.per_stage) == 12
    viol = O.validate(_tuples(tr), _oracle_w(w), slack=SLACK, clock="wall", scale=1.0)
    assert not viol, viol[:5]


def test_interleaved_chunks_and_jitter_valid():
    spec = P.GeneratorSpec(num_stages=3, num_microbatches=4, num_chunks=2,
                           forward=P.uniform(100, 200), backward=P.uniform(100, 200),
                           comm_delay=P.CommDelay(kind="uniform", lo=5, hi=40, seed=3))
    w = P.generate_workload(spec, 6)
    jit = P.JITTER_PRESETS["J1"]
    tr, m = run_gpu(w, "bf", 4, time_scale=0.1, seed=6, jitter=jit)
    inj = O.injection_table(_oracle_w(w), "J1", 6)
    viol = O.validate(_tuples(tr), _oracle_w(w), inj, slack=SLACK, clock="wall", scale=0.1)
    assert not viol, viol[:5]


def test_tp_order_identical_across_ranks():
    spec = P.GeneratorSpec(num_stages=3, num_microbatches=6, tp_group_size=2,
                           forward=P.uniform(100, 300), backward=P.uniform(100, 300))
    w = P.generate_workload(spec, 7)
    tp = P.TpGroup(group_size=2, coordination_round_cost=5, skew_lo=0, skew_hi=60)
    tr, m = run_gpu(w, "bf", 32, time_scale=1.0, seed=7, tp=tp)
    assert len(tr.execs()) == 2 * w.task_count()
    for s in range(3):
        seqs = [[(e.direction, e.microbatch) for e in sorted(tr.execs(rank=r), key=lambda e: e.t_start)
                 if e.stage == s] for r in (0, 1)]
        assert seqs[0] == seqs[1]
    assert m.agreed_rounds > 0


def test_watchdog_fires_on_impossible_schedule():
    # a fixed order whose heads wait on each other (B before its F) never finishes
    w = P.generate_workload(_spec(2, 2), 0)
    bad = P.FixedSchedule(tuple(
        tuple(sorted(st, key=lambda t: t.direction)) for st in P.build_1f1b_schedule(w).per_stage_order))
    from paper_2605_18750_b200.runtime import LiveWatchdogError
    with pytest.raises(LiveWatchdogError):
        run_gpu(w, "bf", 32, time_scale=1.0, mode="fixed", schedule=bad, watchdog_secs=2)


def test_zb_h1_fixed_schedule_on_lanes():
    """A ZB-H1-like FixedSchedule (W tasks deferred into the cool-down) on the
    free-running lanes in FIXED mode: per-stage order followed, trace valid."""
    w = P.generate_workload(_spec(4, 8, decompose_backward=True), 9)
    sched = P.build_zb_h1_schedule(w)
    tr, m = run_gpu(w, "bfw", 32, time_scale=1.0, seed=9, mode="fixed", schedule=sched)
    want = [[(t.direction, t.microbatch, t.chunk) for t in st] for st in sched.per_stage_order]
    assert _seqs(tr, 4) == want
    viol = O.validate(_tuples(tr), _oracle_w(w), slack=SLACK, clock="wall", scale=1.0)
    assert not viol, viol[:5]


def test_external_hint_replay_bit_exact():
    """External ranked hint (arbitration.py:259-278, config hint "file:...") on
    the lanes in replay mode: the oracle's per-stage order."""
    w = P.generate_workload(_spec(4, 8), 11)
    hint = P.HintOrder(kind="external", ranked=(("B", "asc"), ("F", "asc")))
    tr, _ = run_gpu(w, hint, 32, time_scale=1.0, seed=11, mode="replay")
    ev, _ = O.run_rrfp(_oracle_w(w), "external", 32, 11, "J0", ranked=(("B", "asc"), ("F", "asc")))
    want = [[(d, mb, c) for d, mb, c, _, _ in s] for s in O.exec_sequences(ev, 4)]
    assert _seqs(tr, 4) == want


def _golden_wide():
    from golden_util import engine_cases
    return [c for c in engine_cases() if c["name"].startswith(("wide-", "pp8-")) and "deadlock" not in c]


@pytest.mark.parametrize("case", _golden_wide(), ids=lambda c: c["name"])
def test_wide_golden_cases_on_lanes(case):
    """More than 32 microbatches (multi-word ready bitmasks), limits below M,
    TP=2 with 100 microbatches, C=3 external hints: the device lanes replay the
    reference's per-stage order exactly, and free-running they produce a valid
    wall trace."""
    w = P.generate_workload(P.GeneratorSpec.from_json(case["spec"]), case["seed"])
    hint = (P.HintOrder("external", tuple(tuple(e) for e in case["ranked"]))
            if case["hint"] == "external" else P.HintOrder(case["hint"]))
    tp = None
    if case["tp"]:
        tp = P.TpGroup(group_size=w.tp_group_size, coordination_round_cost=case["tp"]["cost"],
                       skew_lo=case["tp"]["skew_lo"], skew_hi=case["tp"]["skew_hi"])
    jit = P.JITTER_PRESETS[case["jitter"]]
    scale = min(1.0, 20000.0 / case["metrics"]["makespan"])    # ~20 ms of device time
    tr, _ = run_gpu(w, hint, case["limit"], time_scale=scale, seed=case["seed"], jitter=jit, tp=tp,
                    mode="replay")
    want = [[(d, mb, c) for d, mb, c, _, _ in s] for s in case["exec"]["0"]]
    assert _seqs(tr, w.num_stages, 0) == want
    tr, m = run_gpu(w, hint, case["limit"], time_scale=scale, seed=case["seed"], jitter=jit, tp=tp)
    assert m.total_tasks == w.task_count()
    viol = [v for v in O.validate(_tuples(tr), _oracle_w(w), slack=SLACK, clock="wall", scale=scale)
            if v[0] != "duration"]
    assert not viol, viol[:5]


# ---------------------------------------------------------------- replay mode
def _case_inputs(case):
    w = P.generate_workload(P.GeneratorSpec.from_json(case["spec"]), case["seed"])
    hint = (P.HintOrder("external", tuple(tuple(e) for e in case["ranked"]))
            if case["hint"] == "external" else P.HintOrder(case["hint"]))
    tp = None
    if case["tp"]:
        tp = P.TpGroup(group_size=w.tp_group_size, coordination_round_cost=case["tp"]["cost"],
                       skew_lo=case["tp"]["skew_lo"], skew_hi=case["tp"]["skew_hi"])
    return w, hint, tp


MAX_LANES = 16   # lanes of one process = spinning conditional graphs; beyond ~16 per
                 # process they share hardware queues (CUDA_DEVICE_MAX_CONNECTIONS <= 32)


def _lanes(case):
    sp = case["spec"]
    return sp.get("num_stages", 1) * (sp.get("tp_group_size") or 1)


def _all_cases():
    from golden_util import engine_cases
    return [c for c in engine_cases() if _lanes(c) <= MAX_LANES]


@pytest.mark.parametrize("case", _all_cases(), ids=lambda c: c["name"])
def test_replay_lanes_reproduce_reference_engine(case):
    """North-star parity on the DEVICE DISPATCHER: every lane decides with its
    own arbiter (and K4 round for TP) at the reference engine's virtual times,
    learning about other stages only through its inbox; the resulting trace
    equals run_rrfp's event for event (exec / send / recv / coord / block, all
    virtual start/end times), the metrics are identical, and the deadlock
    cases raise EngineDeadlockError."""
    w, hint, tp = _case_inputs(case)
    jit = P.JITTER_PRESETS[case["jitter"]]
    scale = min(1.0, 20000.0 / max(1, case.get("metrics", {}).get("makespan", 20000)))
    if "deadlock" in case:
        with pytest.raises(P.EngineDeadlockError):
            run_gpu(w, hint, case["limit"], time_scale=scale, seed=case["seed"], jitter=jit, tp=tp,
                    mode="replay", watchdog_secs=60)
        return
    tr, m = run_gpu(w, hint, case["limit"], time_scale=scale, seed=case["seed"], jitter=jit, tp=tp,
                    mode="replay", watchdog_secs=60)
    assert tr.clock == "virtual"
    norm = lambda e: tuple(-1 if v is None else v for v in e)
    got = sorted(norm(e.to_json().values()) for e in tr.events)
    want = sorted(norm(e) for e in case["events"])
    assert got == want
    assert m.to_json() == case["metrics"]


def test_replay_lanes_fixed_schedule_matches_run_fixed():
    """Replay + a FixedSchedule: the lanes' head-blocking 1F1B under the
    virtual clock equals baselines.run_fixed (golden fixed_exec)."""
    from golden_util import engine_cases
    for case in [c for c in engine_cases() if c.get("fixed")][:6]:
        w, hint, tp = _case_inputs(case)
        if w.tp_group_size > 1:
            continue
        jit = P.JITTER_PRESETS[case["jitter"]]
        tr, fm = run_gpu(w, "bf", 1 << 20, time_scale=0.01, seed=case["seed"], jitter=jit,
                         mode="replay", schedule=P.build_1f1b_schedule(w), watchdog_secs=60)
        per = [[] for _ in range(w.num_stages)]
        for e in sorted(tr.execs(), key=lambda e: (e.t_start, e.t_end)):
            per[e.stage].append([e.direction, e.microbatch, e.chunk, e.t_start, e.t_end])
        assert per == case["fixed_exec"], case["name"]
        assert fm.makespan == case["fixed_metrics"]["makespan"]


# ------------------------------------------------- free-mode decision oracle
from decision_check import check_decisions


FREE_CASES = ["config1-J0-s0", "config1-J3-s1", "pp8-m32-bfw", "interleaved-tp", "rand31"]


@pytest.mark.parametrize("name", FREE_CASES)
def test_free_mode_decisions_match_oracle(name):
    """Every arbitration the free-running lanes evaluate (ready bitmasks built
    by ballot from the inbox flags, backpressure, phase, admission) is logged
    on the device and re-evaluated with the reference's arbitrate: 100 % match."""
    from golden_util import case_by_name
    case = case_by_name(name)
    w, hint, tp = _case_inputs(case)
    scale = min(1.0, 20000.0 / case["metrics"]["makespan"])
    log = []
    tr, m = run_gpu(w, hint, case["limit"], time_scale=scale, seed=case["seed"],
                    jitter=P.JITTER_PRESETS[case["jitter"]], tp=tp, declog=log, watchdog_secs=60)
    assert len(tr.execs()) == w.task_count() * w.tp_group_size
    n_commit = sum(1 for d in log if d["kind"] != "wait")
    assert n_commit >= w.task_count() * w.tp_group_size - sum(s.n_w for s in m.per_stage) * 0, n_commit
    ranked = tuple(tuple(e) for e in case.get("ranked") or ())
    bad = check_decisions(log, w, hint, case["limit"], ranked)
    assert not bad, bad[:3]


def test_replay_decisions_match_oracle():
    """The replay lanes' log too (virtual-time decisions, every rank)."""
    from golden_util import case_by_name
    case = case_by_name("interleaved-tp")
    w, hint, tp = _case_inputs(case)
    log = []
    run_gpu(w, hint, case["limit"], time_scale=0.01, seed=case["seed"],
            jitter=P.JITTER_PRESETS[case["jitter"]], tp=tp, mode="replay", declog=log)
    assert len(log) >= 750 * 0 + w.task_count()
    assert not check_decisions(log, w, hint, case["limit"])


def test_dispatcher_profile_records_every_step():
    """rrfp_runtime_profile: one record per lane_step_kernel run (every task's
    decision plus the exiting step), stamps ordered entry <= completion done <=
    decision, kinds of the dispatched tasks match the trace; disabling stops it."""
    from paper_2605_18750_b200.runtime import LaneGroup, dispatcher_profile
    w = P.generate_workload(_spec(n=2, m=8), 5)
    g = LaneGroup(w, "bf", 32, 1.0, seed=5)
    try:
        g.run_iteration(30.0)
        g.enable_profile(1024)
        events, t0s = g.run_iteration(30.0)
        prof = g.profile()
        assert len(prof) == 2
        for lane, r in prof.items():
            assert len(r) == w.task_count() // 2 + 1
            r = r.astype("int64")
            assert (r[:, 0] <= r[:, 1]).all() and (r[:, 1] <= r[:, 2]).all()
            kinds = sorted(int(k) for k in (r[:, 3] >> 32))
            assert kinds.count(3) == 1                       # the exiting step
            assert kinds.count(0) == kinds.count(1) == 8     # B and F of every microbatch
        s = dispatcher_profile(prof)
        assert s["complete_us"]["n"] == w.task_count() + 2
        g.enable_profile(0)
        g.run_iteration(30.0)
        assert all(len(r) == 0 for r in g.profile().values())
    finally:
        g.close()
