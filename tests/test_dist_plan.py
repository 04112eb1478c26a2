"""Multi-process host logic (one stage per process) on CPU with gloo, world_size 2:
topology plan, handle exchange and identical replay schedules on every rank."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2605_18750_b200 as P
    from paper_2605_18750_b200.distributed import plan_peers
    from paper_2605_18750_b200 import tables
    peers = plan_peers(rank, world)
    fake = {"stage": rank, "fwd": bytes([rank + 1]) * 64 if rank > 0 else None,
            "bwd": bytes([rank + 11]) * 64 if rank < world - 1 else None}
    allh = [None] * world
    dist.all_gather_object(allh, fake)
    opened = {}
    if peers["writes_fwd_mailbox"]:
        opened["fwd"] = allh[rank + 1]["fwd"]
    if peers["writes_bwd_mailbox"]:
        opened["bwd"] = allh[rank - 1]["bwd"]
    # every rank lowers the same workload independently -> identical tables / schedules
    spec = P.GeneratorSpec(num_stages=world, num_microbatches=8, forward=P.uniform(50, 150),
                           backward=P.uniform(80, 200))
    w = P.generate_workload(spec, 5)
    tr, m = P.run_rrfp(w, "bf", 32, 5, jitter=P.JITTER_PRESETS["J2"], device="cpu")
    order = [(e.stage, e.direction, e.microbatch, e.t_start) for e in tr.execs()]
    tb = tables.lower(w, P.HintOrder("bf"), 32, 5, P.JITTER_PRESETS["J2"])
    allo = [None] * world
    dist.all_gather_object(allo, (order, int(tb.dur.sum()), int(tb.comm.sum())))
    q.put((rank, peers, opened, allo[0] == allo[-1]))
    dist.destroy_process_group()


def test_two_process_plan_and_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    r0, r1 = res
    assert r0[1]["fwd"] == [(1, 0)] and r0[1]["writes_fwd_mailbox"] and not r0[1]["writes_bwd_mailbox"]
    assert r1[1]["bwd"] == [(0, 0)] and r1[1]["writes_bwd_mailbox"] and not r1[1]["writes_fwd_mailbox"]
    assert r0[2]["fwd"] == bytes([2]) * 64      # rank 0 writes into rank 1's F mailbox
    assert r1[2]["bwd"] == bytes([11]) * 64     # rank 1 writes into rank 0's B mailbox
    assert r0[3] and r1[3]                      # identical schedules/tables on both ranks


def test_plan_wraps_for_interleaved_chunks():
    from paper_2605_18750_b200.distributed import plan_peers
    p = plan_peers(3, 4, 2)
    assert p["fwd"] == [(0, 0), (0, 1)] and p["bwd"] == [(2, 0), (2, 1)]
    assert not p["writes_fwd_mailbox"] and p["writes_bwd_mailbox"]


def test_stage_coords_tp_groups():
    """torchrun rank -> (stage, TP rank): TP ranks of a stage are adjacent (config 3: TP2 x PP4)."""
    from paper_2605_18750_b200.distributed import stage_coords
    assert [stage_coords(g, 8, 2) for g in range(8)] == [(s, r, 4) for s in range(4) for r in range(2)]
    assert [stage_coords(g, 4, 1)[:2] for g in range(4)] == [(g, 0) for g in range(4)]
    with pytest.raises(ValueError):
        stage_coords(0, 6, 4)


def test_balanced_layer_split():
    """Layer split against the last stage's LM head (bench --head-cost): every
    layer exactly once, contiguous, and the max stage cost is minimal."""
    from paper_2605_18750_b200.model import split_layers
    for L, N, h in [(24, 8, 1.4), (24, 4, 1.4), (24, 2, 1.4), (32, 4, 1.4), (7, 3, 2.0), (24, 8, 0.0)]:
        parts = [split_layers(L, N, s, h) for s in range(N)]
        assert [i for p in parts for i in p] == list(range(L))
        cost = [len(p) + (h if s == N - 1 else 0) for s, p in enumerate(parts)]
        even = [len(split_layers(L, N, s)) + (h if s == N - 1 else 0) for s in range(N)]
        assert max(cost) <= max(even)
    assert [len(split_layers(24, 8, s, 1.4)) for s in range(8)] == [4, 3, 3, 3, 3, 3, 3, 2]


def test_half_layer_split_is_optimal_and_contiguous():
    """split_units('half'): contiguous, covers every (layer, half) once, and its
    bottleneck equals the brute-force optimum over all cut placements."""
    import itertools
    from paper_2605_18750_b200.model import split_units
    a = 0.42
    w = {"full": 1.0, "attn": a, "mlp": 1 - a}
    for L, N, h in [(4, 3, 1.4), (4, 3, 0.0), (5, 4, 1.4), (6, 4, 0.7), (3, 5, 1.4)]:
        parts = [split_units(L, N, s, h, "half", a) for s in range(N)]
        flat = []
        for p in parts:
            assert p, "empty stage"
            for l, pt in p:
                flat += [(l, "attn"), (l, "mlp")] if pt == "full" else [(l, pt)]
        assert flat == [(l, pt) for l in range(L) for pt in ("attn", "mlp")]
        got = max(sum(w[pt] for _, pt in p) + (h if s == N - 1 else 0) for s, p in enumerate(parts))
        cost = [a if i % 2 == 0 else 1 - a for i in range(2 * L)]
        best = min(max(sum(cost[b[i]:b[i + 1]]) + (h if i == N - 1 else 0) for i in range(N))
                   for cuts in itertools.combinations(range(1, 2 * L), N - 1)
                   for b in [(0, *cuts, 2 * L)])
        assert abs(got - best) < 1e-9, (L, N, h, got, best)
    # 1.3B at PP=8: 3.58 layer-equivalents at the bottleneck instead of 4.0
    costs = [sum(w[pt] for _, pt in split_units(24, 8, s, 1.4, "half", a)) + (1.4 if s == 7 else 0)
             for s in range(8)]
    assert abs(max(costs) - 3.58) < 1e-9
    assert [l for l, _ in split_units(24, 8, 0, 1.4, "layer")] == [0, 1, 2, 3]
