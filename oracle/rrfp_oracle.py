"""CPU oracle for the RRFP hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-Python/numpy restatement of the reference
scheduling algorithm (arXiv 2605.18750, package ``rrfp`` under
/root/reference/pkg/src/rrfp).  It exists so the tests, ``smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg can check and
time the B200 path against the reference semantics.  The product package
(``paper_2605_18750_b200``) never imports it; the product path fails loudly
if its CUDA library is missing.

Parity pinning: every function below was checked against the real
reference (imported read-only in the build container) through the golden
fixtures in ``tests/golden/`` produced by ``oracle/gen_golden.py``
(dispatch traces, makespans, injection tables, comm-delay tables,
arbitration snapshots).  The RNG is numpy's PCG64 seeded from a blake2b
digest of the label path, exactly as the reference's ``rng.substream``
(rng.py:19-36); numpy 2.3.x is the version the fixtures were made with.

Representation (deliberately different from the reference's classes):
a task is the tuple ``(d, s, mb, c)`` with ``d`` in "F"/"B"/"W"; a workload
is a plain dict; traces are lists of 8-tuples
``(t0, t1, stage, rank, mb, chunk, dir, kind)``.
"""

from __future__ import annotations

import hashlib
import heapq
import math
import queue
import threading
import time

import numpy as np

F, B, W = "F", "B", "W"
_DIR_ORDER = {B: 0, F: 1, W: 2}          # workload.py:37-40 (tie-break rank)
COMM_KINDS = ("InterStageForward", "InterStageBackward", "ChunkWrap")


def task_key(t):
    d, s, mb, c = t
    return f"{d}:{s}:{mb}:{c}"


def parse_key(k):
    d, s, mb, c = k.split(":")
    return (d, int(s), int(mb), int(c))


# ---------------------------------------------------------------- RNG -----
def substream(seed, *labels):
    """rng.py:19-36 -- blake2b(16) over "seed/label/label..." -> PCG64."""
    h = hashlib.blake2b(digest_size=16)
    h.update(str(int(seed)).encode())
    for lab in labels:
        h.update(b"/" + str(lab).encode())
    return np.random.Generator(np.random.PCG64(int.from_bytes(h.digest(), "big")))


def _lognormal_clamped(rng, mu, sigma, lo, hi):
    """workload.py:134-141 -- rejection sample, clamp after 1000 tries."""
    v = lo
    for _ in range(1000):
        v = int(round(float(np.exp(rng.normal(mu, sigma)))))
        if lo <= v <= hi:
            return v
    return min(max(v, lo), hi)


def sample_dist(dist, rng):
    """DistSpec.sample, workload.py:333-338."""
    kind = dist["kind"]
    if kind == "constant":
        return dist["value"]
    if kind == "uniform":
        return int(rng.integers(dist["lo"], dist["hi"] + 1))
    return _lognormal_clamped(rng, dist["mu"], dist["sigma"], dist["lo"], dist["hi"])


def comm_delay_sample(comm, src, dst, kind):
    """CommDelay.sample, workload.py:109-117 (keyed by the edge itself)."""
    if kind not in COMM_KINDS:
        return 0
    ck = comm.get("kind", "constant")
    if ck == "constant":
        return comm.get("value", 0)
    rng = substream(comm.get("seed", 0), "comm", task_key(src), task_key(dst))
    if ck == "uniform":
        return int(rng.integers(comm["lo"], comm["hi"] + 1))
    return _lognormal_clamped(rng, comm["mu"], comm["sigma"], comm["lo"], comm["hi"])


# ----------------------------------------------------------- workload -----
def generate(spec, seed):
    """generate_workload, workload.py:417-463.

    ``spec`` is a GeneratorSpec JSON dict; returns the workload dict
    {N, M, C, R, lat: {task: us}, comm, dec, beta}.
    """
    n, m, cc = spec["num_stages"], spec["num_microbatches"], spec.get("num_chunks", 1)
    heavy_last = spec.get("heavy_last", 1.0)
    heavy_prefix = spec.get("heavy_prefix", 1.0)
    prefix = -(-n // 4)
    lat = {}
    for s in range(n):
        for d, dist in ((F, spec["forward"]), (B, spec["backward"])):
            rng = substream(seed, "lat", d, s)
            for c in range(cc):
                for mb in range(m):
                    v = sample_dist(dist, rng)
                    if s == n - 1 and heavy_last != 1.0:
                        v = int(round(v * heavy_last))
                    if d == F and s < prefix and heavy_prefix != 1.0:
                        v = int(round(v * heavy_prefix))
                    lat[(d, s, mb, c)] = max(v, 1)
    dec = bool(spec.get("decompose_backward", False))
    beta = spec.get("backward_split_fraction", 0.5)
    if dec:
        for s in range(n):
            for mb in range(m):
                for c in range(cc):
                    full = lat[(B, s, mb, c)]
                    part = int(round(beta * full))
                    lat[(B, s, mb, c)] = part
                    lat[(W, s, mb, c)] = full - part
    comm = dict(spec.get("comm_delay", {"kind": "constant", "value": 0}))
    if comm.get("kind", "constant") != "constant" and comm.get("seed", 0) == 0:
        comm["seed"] = seed
    return {"N": n, "M": m, "C": cc, "R": spec.get("tp_group_size", 1), "lat": lat,
            "comm": comm, "dec": dec, "beta": beta}


def from_workload_json(obj):
    """Workload.from_json, workload.py:205-216."""
    return {"N": obj["num_stages"], "M": obj["num_microbatches"], "C": obj["num_chunks"],
            "R": obj.get("tp_group_size", 1),
            "lat": {parse_key(k): int(v) for k, v in obj["latency"].items()},
            "comm": obj.get("comm_delay", {"kind": "constant", "value": 0}),
            "dec": obj.get("decompose_backward", False),
            "beta": obj.get("backward_split_fraction", 0.5)}


def task_graph(w):
    """build_task_graph, workload.py:234-260 -> list of (src, dst, kind)."""
    n, m, cc = w["N"], w["M"], w["C"]
    out = []
    for mb in range(m):
        for c in range(cc):
            for s in range(n):
                f, b = (F, s, mb, c), (B, s, mb, c)
                if s > 0:
                    out.append(((F, s - 1, mb, c), f, "InterStageForward"))
                elif c > 0:
                    out.append(((F, n - 1, mb, c - 1), f, "ChunkWrap"))
                if s < n - 1:
                    out.append(((B, s + 1, mb, c), b, "InterStageBackward"))
                elif c < cc - 1:
                    out.append(((B, 0, mb, c + 1), b, "ChunkWrap"))
                out.append((f, b, "LocalForwardToBackward"))
                if w["dec"]:
                    out.append((b, (W, s, mb, c), "BackwardToWeight"))
    return out


def route(w, t):
    """Destination of a finished task's output: engine.py:181-209 / live.py:186-199.

    Returns (dst_task, edge_kind), "turnaround" or None (gradient exits).
    """
    d, s, mb, c = t
    n, cc = w["N"], w["C"]
    if d == F:
        if s < n - 1:
            return (F, s + 1, mb, c), "InterStageForward"
        if c < cc - 1:
            return (F, 0, mb, c + 1), "ChunkWrap"
        return "turnaround"
    if s > 0:
        return (B, s - 1, mb, c), "InterStageBackward"
    if c > 0:
        return (B, n - 1, mb, c - 1), "ChunkWrap"
    return None


# ------------------------------------------------------------- jitter -----
JITTER = {  # jitter.py:55-60
    "J0": (0.0, 0, 0.0), "J1": (0.1, 5000, 0.5),
    "J2": (0.2, 10000, 1.0), "J3": (0.3, 15000, 1.5),
}


def jitter_cfg(level_or_obj):
    if isinstance(level_or_obj, str):
        p, base, scale = JITTER[level_or_obj]
        return {"probability": p, "base_delay": base, "scale": scale, "level": level_or_obj}
    return dict(level_or_obj)


def ema(prev, c):
    """ema_update, jitter.py:76-80 (integer half-up)."""
    if prev < 0 or c < 0:
        raise ValueError("EMA inputs must be non-negative")
    return (9 * prev + c + 5) // 10


def injection_table(w, cfg, seed):
    """build_injection_table, jitter.py:97-118 (+ sample_delay 83-94)."""
    cfg = jitter_cfg(cfg)
    p, base, scale = cfg["probability"], cfg["base_delay"], cfg["scale"]
    out = {}
    if not (p > 0 and scale > 0):
        return out
    for s in range(w["N"]):
        rng = substream(seed, "jitter", cfg.get("level", "J0"), s)
        e = -1
        for mb in range(w["M"]):
            for c in range(w["C"]):
                for d in (F, B):
                    t = (d, s, mb, c)
                    lat = w["lat"][t]
                    e = lat if e < 0 else ema(e, lat)
                    gate, r = rng.random(), rng.random()
                    if gate < p:
                        v = int(round(scale * max(base, max(e, 0)) * (0.5 + r)))
                        if v:
                            out[t] = v
    return out


# -------------------------------------------------------- arbitration -----
class View:
    """One rank's ready view of one stage (arbitration.py:93-116)."""

    def __init__(self):
        self.fready = set()     # (mb, c)
        self.bready = set()     # (mb, c)
        self.admission = None   # mb of the next chunk-0 forward at stage 0
        self.wpend = None       # shared set of (mb, c), set by the stage

    def fcands(self):
        out = set(self.fready)
        if self.admission is not None:
            out.add((self.admission, 0))
        return out


class StageCtl:
    """bp/arb/progress bundle of one stage (arbitration.py:132-229)."""

    def __init__(self, limit, n_chunks, n_mb):
        self.limit, self.C, self.M = limit, n_chunks, n_mb
        self.nf = self.nb = 0
        self.mode = "normal"
        self.focus = -1
        self.phase = ""
        self.done = set()       # (mb, c, d) for d in F/B

    def finished(self, mb):
        return all((mb, c, d) in self.done for c in range(self.C) for d in (F, B))

    def next_step(self, mb):
        """next_in_completion_order, arbitration.py:174-185."""
        for c in range(self.C):
            if (mb, c, F) not in self.done:
                return (F, mb, c)
        for c in reversed(range(self.C)):
            if (mb, c, B) not in self.done:
                return (B, mb, c)
        return None

    def update_bp(self):
        """update_backpressure, arbitration.py:188-215."""
        if self.nf - self.nb < self.limit:
            self.mode, self.focus = "normal", -1
            return
        if self.C == 1:
            self.mode, self.focus = "drain", -1
            return
        f = self.focus
        if self.mode != "focus" or f < 0 or self.finished(f):
            f = next((j for j in range(self.M) if not self.finished(j)), -1)
            if f < 0:
                self.mode, self.focus = "normal", -1
                return
        self.mode, self.focus = "focus", f


def _pick(cands, key):
    return min(cands, key=key) if cands else None


def arbitrate(view, ctl, hint, dec, ranked=()):
    """arbitrate + _weight_fallback, arbitration.py:232-303.

    Returns ("F"|"B"|"W", (mb, c)) or ("wait", None).  Pure.
    """
    fkey = lambda t: (t[1], t[0])           # smaller chunk, then mb
    bkey = lambda t: (-t[1], t[0])          # larger chunk, then mb
    if ctl.mode == "drain":
        t = _pick(view.bready, bkey)
        return (B, t) if t is not None else ("wait", None)
    if ctl.mode == "focus":
        step = ctl.next_step(ctl.focus)
        if step is None:
            return ("wait", None)
        d, mb, c = step
        pool = view.fcands() if d == F else view.bready
        return (d, (mb, c)) if (mb, c) in pool else ("wait", None)

    def wfallback():
        if dec and view.wpend:
            return (W, _pick(view.wpend, bkey))
        return ("wait", None)

    if hint == "external":
        for d, rule in ranked:
            pool = view.fcands() if d == F else view.bready if d == B else set(view.wpend or ())
            if not pool:
                continue
            if d == F:
                k = fkey if rule == "asc" else bkey
            elif d == B:
                k = bkey if rule == "desc" else fkey
            else:
                k = bkey
            return (d, _pick(pool, k))
        return wfallback()
    if hint == "bprio":
        order = (B, F)
    elif hint == "fprio":
        order = (F, B)
    else:
        first = ctl.phase or (F if hint == "fb" else B)
        order = (first, B if first == F else F)
    for d in order:
        t = _pick(view.bready, bkey) if d == B else _pick(view.fcands(), fkey)
        if t is not None:
            return (d, t)
    return wfallback()


def advance_phase(ctl, hint, kind):
    """advance_round_phase, arbitration.py:306-320."""
    if hint not in ("bf", "fb", "bfw"):
        return
    ctl.phase = F if kind == B else B if kind == F else ""


# ------------------------------------------------------------- engine -----
class DeadlockError(RuntimeError):
    pass


def run_rrfp(w, hint="bf", limit=32, seed=0, jitter="J0", tp=None, ranked=()):
    """Virtual-clock readiness-driven engine, engine.py:93-466.

    tp = {"cost": int, "skew_lo": int, "skew_hi": int} (TpGroup fields).
    Returns (events, metrics) with events as 8-tuples in emission order.
    """
    if limit < 1:
        raise ValueError("buffer_limit must be >= 1")
    n, m, cc, R = w["N"], w["M"], w["C"], w["R"]
    tp = dict({"cost": 5, "skew_lo": 0, "skew_hi": 0}, **(tp or {}))
    inj = injection_table(w, jitter, seed)
    per_stage = m * cc * (3 if w["dec"] else 2)
    views = [[View() for _ in range(R)] for _ in range(n)]
    ctls = [StageCtl(limit, cc, m) for _ in range(n)]
    pend = [[{} for _ in range(R)] for _ in range(n)]   # gated grads per rank
    busy = [0] * n
    coord_until = [0] * n
    awaiting = [False] * n
    remaining = [per_stage] * n
    compute = [0] * n
    coord = [0] * n
    nw = [0] * n
    windows = [[] for _ in range(n)]
    for s in range(n):
        shared = set()
        for v in views[s]:
            v.wpend = shared
    for v in views[0]:
        v.admission = 0
    next_adm = 0
    heap, seq = [], [0]
    ev = []
    occ_open, occ_closed = {}, {}
    stats = {"agreed": 0, "deferred": 0, "done": 0, "clock": 0}

    def push(t, kind, stage, rank, task, payload=None):
        if task is None:
            k = (t, stage, 9, 0, 0, rank, seq[0])
        else:
            k = (t, stage, _DIR_ORDER[task[0]], task[2], task[3], rank, seq[0])
        seq[0] += 1
        heapq.heappush(heap, (k, kind, stage, rank, task, payload))

    def emit(kind, t0, t1, stage, rank, task):
        if task is None:
            ev.append((t0, t1, stage, rank, None, None, None, kind))
        else:
            ev.append((t0, t1, stage, rank, task[2], task[3], task[0], kind))

    def occ_on(s, buf, r, key, t):
        occ_open.setdefault((s, buf, r), {})[key] = t

    def occ_off(s, buf, r, key, t):
        o = occ_open.get((s, buf, r), {}).pop(key, None)
        if o is not None:
            occ_closed.setdefault((s, buf, r), []).append((o, t))

    def send(task, end):                     # engine.py:181-221
        s = task[1]
        dst = route(w, task)
        if dst == "turnaround":
            mb, c = task[2], task[3]
            for r in range(R):
                views[s][r].bready.add((mb, c))
                occ_on(s, "backward_ready", r, (B, s, mb, c), end)
            return
        if dst is None:
            return
        dtask, kind = dst
        buf = "forward_finished" if task[0] == F else "backward_finished"
        deliver = end + comm_delay_sample(w["comm"], task, dtask, kind)
        occ_on(s, buf, 0, (task, dtask), end)
        push(deliver, "release", s, 0, None, (buf, (task, dtask)))
        emit("send", end, deliver, s, None, task)
        for r in range(R):
            sk = 0
            if tp["skew_hi"] > 0 and R > 1:
                sk = int(substream(seed, "skew", task_key(dtask), r).integers(
                    tp["skew_lo"], tp["skew_hi"] + 1))
            push(deliver + sk, "arrival", dtask[1], r, dtask)

    def on_arrival(t, s, r, task):           # engine.py:225-238
        awaiting[s] = False
        mb, c = task[2], task[3]
        if task[0] == F:
            views[s][r].fready.add((mb, c))
            occ_on(s, "forward_ready", r, task, t)
        elif (mb, c, F) in ctls[s].done:
            views[s][r].bready.add((mb, c))
            occ_on(s, "backward_ready", r, task, t)
        else:
            pend[s][r][task] = t
        emit("recv", t, t, s, r, task)

    def on_complete(t, s, task):             # engine.py:240-266
        d, _, mb, c = task
        ctl = ctls[s]
        if d != W:
            ctl.done.add((mb, c, d))
        remaining[s] -= 1
        stats["done"] += 1
        if d == F:
            ctl.nf += 1
            bt = (B, s, mb, c)
            for r in range(R):
                if pend[s][r].pop(bt, None) is not None:
                    views[s][r].bready.add((mb, c))
                    occ_on(s, "backward_ready", r, bt, t)
            send(task, t)
        elif d == B:
            ctl.nb += 1
            for r in range(R):
                occ_off(s, "forward_ready", r, (F, s, mb, c), t)
                occ_off(s, "backward_ready", r, task, t)
            if w["dec"]:
                views[s][0].wpend.add((mb, c))
            send(task, t)
        else:
            nw[s] += 1

    def commit(s, kind, mc, start):          # engine.py:270-296
        nonlocal next_adm
        mb, c = mc
        task = (kind, s, mb, c)
        dur = w["lat"][task] + inj.get(task, 0)
        if kind == F:
            if views[s][0].admission is not None and (views[s][0].admission, 0) == mc and s == 0:
                next_adm += 1
                for v in views[s]:
                    v.admission = next_adm if next_adm < m else None
            else:
                for v in views[s]:
                    v.fready.discard(mc)
        elif kind == B:
            for v in views[s]:
                v.bready.discard(mc)
        else:
            views[s][0].wpend.discard(mc)
        advance_phase(ctls[s], hint, kind)
        busy[s] = start + dur
        compute[s] += dur
        windows[s].append((start, start + dur))
        for r in range(R):
            emit("exec", start, start + dur, s, r if R > 1 else None, task)
        push(start + dur, "complete", s, 0, task)

    def dispatch(s, now):                    # engine.py:298-340
        if busy[s] > now or coord_until[s] > now or remaining[s] == 0:
            return
        ctl = ctls[s]
        ctl.update_bp()
        ds = [arbitrate(views[s][r], ctl, hint, w["dec"], ranked) for r in range(R)]
        if R == 1:
            if ds[0][0] == "wait":
                ctl.phase = ""
                return
            commit(s, ds[0][0], ds[0][1], now)
            return
        if all(d[0] == "wait" for d in ds):
            ctl.phase = ""
            return
        if all(d[0] == W for d in ds):
            commit(s, W, ds[0][1], now)
            return
        if awaiting[s]:
            return
        props = [(d[0], d[1]) if d[0] in (F, B) else None for d in ds]
        cost = tp["cost"]
        coord[s] += cost
        windows[s].append((now, now + cost))
        if props[0] is not None and all(p == props[0] for p in props):
            stats["agreed"] += 1
            k, mc = props[0]
            emit("coord", now, now + cost, s, None, (k, s, mc[0], mc[1]))
            commit(s, k, mc, now + cost)
        else:
            stats["deferred"] += 1
            emit("coord", now, now + cost, s, None, None)
            coord_until[s] = now + cost
            awaiting[s] = True
            ctl.phase = ""
            push(now + cost, "coord_end", s, 0, None)

    for s in range(n):
        dispatch(s, 0)
    while heap:
        tick = heap[0][0][0]
        touched = set()
        while heap and heap[0][0][0] == tick:
            _, kind, s, r, task, payload = heapq.heappop(heap)
            if kind == "complete":
                on_complete(tick, s, task)
            elif kind == "arrival":
                on_arrival(tick, s, r, task)
            elif kind == "release":
                occ_off(s, payload[0], 0, payload[1], tick)
            touched.add(s)
        stats["clock"] = tick
        for s in sorted(touched):
            dispatch(s, tick)
    total = n * per_stage
    if stats["done"] != total:
        raise DeadlockError(f"quiescent with {total - stats['done']} unfinished tasks")
    makespan = stats["clock"]
    per = []
    for s in range(n):
        occ = {}
        for buf in ("forward_ready", "forward_finished", "backward_ready", "backward_finished"):
            worst = 0
            for r in range(R):
                ivs = list(occ_closed.get((s, buf, r), []))
                ivs += [(t, makespan) for t in occ_open.get((s, buf, r), {}).values()]
                worst = max(worst, _max_overlap(ivs))
            occ[buf] = worst
        per.append({"stage": s, "compute": compute[s], "blocking": makespan - compute[s] - coord[s],
                    "tp_coord": coord[s], "n_f": ctls[s].nf, "n_b": ctls[s].nb, "n_w": nw[s],
                    "max_occupancy": occ})
        for g in gaps(windows[s], makespan):
            ev.append((g[0], g[1], s, None, None, None, None, "block"))
    metrics = {"makespan": makespan, "total_tasks": total, "agreed_rounds": stats["agreed"],
               "deferred_rounds": stats["deferred"], "per_stage": per}
    return ev, metrics


def _max_overlap(ivs):
    """engine.py:417-430."""
    marks = []
    for a, b in ivs:
        marks.append((a, 1))
        marks.append((max(a, b), -1))
    marks.sort()
    cur = peak = 0
    for _, dlt in marks:
        cur += dlt
        peak = max(peak, cur)
    return peak


def gaps(windows, horizon):
    """engine._gaps, engine.py:433-449."""
    out, prev = [], 0
    merged = []
    for a, b in sorted(windows):
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    for a, b in merged:
        if a > prev:
            out.append((prev, a))
        prev = max(prev, b)
    if prev < horizon:
        out.append((prev, horizon))
    return out


# ---------------------------------------------------------- baselines -----
def one_f_one_b(w):
    """build_1f1b_schedule, baselines.py:68-91 -> per-stage task lists."""
    if w["C"] != 1:
        raise ValueError("1F1B baseline covers non-interleaved workloads only")
    if w["dec"]:
        raise ValueError("1F1B baseline does not decompose backward")
    n, m = w["N"], w["M"]
    out = []
    for s in range(n):
        warm = min(m, n - 1 - s)
        seq = [(F, s, j, 0) for j in range(warm)]
        nf, nb = warm, 0
        while nf < m:
            seq += [(F, s, nf, 0), (B, s, nb, 0)]
            nf, nb = nf + 1, nb + 1
        seq += [(B, s, j, 0) for j in range(nb, m)]
        out.append(seq)
    return out


def run_fixed(order, w, injected=None):
    """run_fixed, baselines.py:94-172: start = max(stage clock, pred arrivals)."""
    injected = injected or {}
    preds = {}
    for src, dst, kind in task_graph(w):
        preds.setdefault(dst, []).append((src, comm_delay_sample(w["comm"], src, dst, kind)))
    n = w["N"]
    head, clock, end = [0] * n, [0] * n, {}
    comp = [0] * n
    ev, win = [], [[] for _ in range(n)]
    total = sum(len(o) for o in order)
    done = 0
    while done < total:
        moved = False
        for s in range(n):
            while head[s] < len(order[s]):
                t = order[s][head[s]]
                ps = preds.get(t, ())
                if any(p not in end for p, _ in ps):
                    break
                dur = w["lat"][t] + injected.get(t, 0)
                st = max([clock[s]] + [end[p] + dl for p, dl in ps])
                end[t] = clock[s] = st + dur
                comp[s] += dur
                win[s].append((st, st + dur))
                ev.append((st, st + dur, s, None, t[2], t[3], t[0], "exec"))
                head[s] += 1
                done += 1
                moved = True
        if not moved:
            raise DeadlockError("schedule-induced deadlock")
    mk = max(end.values()) if end else 0
    per = []
    for s in range(n):
        per.append({"stage": s, "compute": comp[s], "blocking": mk - comp[s], "tp_coord": 0,
                    "n_f": sum(1 for t in order[s] if t[0] == F),
                    "n_b": sum(1 for t in order[s] if t[0] == B), "n_w": 0, "max_occupancy": {}})
        prev = 0
        for a, b in sorted(win[s]):
            if a > prev:
                ev.append((prev, a, s, None, None, None, None, "block"))
            prev = max(prev, b)
        if prev < mk:
            ev.append((prev, mk, s, None, None, None, None, "block"))
    return ev, {"makespan": mk, "total_tasks": total, "agreed_rounds": 0, "deferred_rounds": 0,
                "per_stage": per}


# ------------------------------------------------------ trace helpers -----
def exec_sequences(events, n_stages, rank=0):
    """Per-stage list of (d, mb, c, t0, t1) exec events for one rank."""
    seqs = [[] for _ in range(n_stages)]
    for t0, t1, s, r, mb, c, d, kind in events:
        if kind == "exec" and (r is None or r == rank):
            seqs[s].append((d, mb, c, t0, t1))
    return seqs


def dispatch_hash(events, n_stages):
    """SURVEY.md App. B canonical dispatch hash."""
    seqs = exec_sequences(events, n_stages)
    text = "\n".join(" ".join(f"{d}:{mb}:{c}@{a}-{b}" for d, mb, c, a, b in seq) for seq in seqs)
    return hashlib.sha256(text.encode()).hexdigest()[:16]


# ---------------------------------------------------------------- live -----
def run_live(w, hint="bf", limit=32, time_scale=1.0, seed=0, jitter="J0", tp=None,
             watchdog_secs=30.0, ranked=()):
    """Wall-clock threaded executor restated from live.py:111-523.

    3 threads per (stage, rank): compute worker, sender, receiver, over
    bounded queues (cap = limit + C); tasks are timed sleeps/spins of
    latency * time_scale.  TP rounds resolve atomically under the stage
    lock (live.py:246-277).  Used as the CPU baseline arm.
    Returns (events, makespan_us).
    """
    n, m, cc, R = w["N"], w["M"], w["C"], w["R"]
    tp = dict({"cost": 5, "skew_lo": 0, "skew_hi": 0}, **(tp or {}))
    inj = injection_table(w, jitter, seed)
    cap = limit + cc
    per_stage = m * cc * (3 if w["dec"] else 2)
    poll = 0.02
    stop = threading.Event()
    ev_lock = threading.Lock()
    events = []
    t_epoch = time.perf_counter_ns()
    now_us = lambda: (time.perf_counter_ns() - t_epoch) // 1000

    def emit(kind, t0, t1, s, r, task):
        with ev_lock:
            events.append((t0, t1, s, r, None if task is None else task[2],
                           None if task is None else task[3],
                           None if task is None else task[0], kind))

    class G:
        pass

    groups = []
    for s in range(n):
        g = G()
        g.lock = threading.Lock()
        g.cv = threading.Condition(g.lock)
        g.views = [View() for _ in range(R)]
        shared = set()
        for v in g.views:
            v.wpend = shared
            if s == 0:
                v.admission = 0
        g.next_adm = 0
        g.ctl = StageCtl(limit, cc, m)
        g.pend = [set() for _ in range(R)]
        g.remaining = per_stage
        g.version = 0
        g.checked = set()
        g.outcome = None
        g.acks = 0
        g.round = 0
        g.finishers = 0
        g.finish_round = 0
        g.sends = []
        groups.append(g)
    out_q = {(s, r): queue.Queue(maxsize=cap) for s in range(n) for r in range(R)}
    in_q = {(s, r): queue.Queue(maxsize=cap) for s in range(n) for r in range(R)}
    progress = [0]
    failure = []

    def spin(us):
        deadline = time.perf_counter_ns() + int(us * 1000)
        while True:
            rem = deadline - time.perf_counter_ns()
            if rem <= 0:
                return
            if rem > 2_000_000:
                time.sleep((rem - 1_000_000) / 1e9)
            elif rem > 300_000:
                time.sleep(0.0001)

    def commit(g, s, kind, mc):
        if kind == F:
            if s == 0 and g.views[0].admission is not None and (g.views[0].admission, 0) == mc:
                g.next_adm += 1
                for v in g.views:
                    v.admission = g.next_adm if g.next_adm < m else None
            else:
                for v in g.views:
                    v.fready.discard(mc)
        elif kind == B:
            for v in g.views:
                v.bready.discard(mc)
        else:
            g.views[0].wpend.discard(mc)
        advance_phase(g.ctl, hint, kind)

    def resolve(g, s):
        g.ctl.update_bp()
        ds = [arbitrate(g.views[r], g.ctl, hint, w["dec"], ranked) for r in range(R)]
        if all(d[0] == "wait" for d in ds):
            g.ctl.phase = ""
            return ("wait", None, 0, g.version)
        if all(d[0] == W for d in ds):
            commit(g, s, W, ds[0][1])
            return ("exec", (W, s) + ds[0][1], 0, g.version)
        props = [(d[0], d[1]) if d[0] in (F, B) else None for d in ds]
        cost = tp["cost"] if R > 1 else 0
        if props[0] is not None and all(p == props[0] for p in props):
            commit(g, s, props[0][0], props[0][1])
            return ("exec", (props[0][0], s) + props[0][1], cost, g.version)
        g.ctl.phase = ""
        return ("defer", None, cost, g.version)

    def complete(g, s, task, t_end):
        d, _, mb, c = task
        if d != W:
            g.ctl.done.add((mb, c, d))
        g.remaining -= 1
        progress[0] += 1
        sends = []
        if d == F:
            g.ctl.nf += 1
            for r in range(R):
                if (mb, c) in g.pend[r]:
                    g.pend[r].discard((mb, c))
                    g.views[r].bready.add((mb, c))
            dst = route(w, task)
            if dst == "turnaround":
                for r in range(R):
                    g.views[r].bready.add((mb, c))
            elif dst is not None:
                sends.append(dst)
        elif d == B:
            g.ctl.nb += 1
            if w["dec"]:
                g.views[0].wpend.add((mb, c))
            dst = route(w, task)
            if dst is not None:
                sends.append(dst)
        g.version += 1
        return sends

    def worker(s, r):
        g = groups[s]
        while not stop.is_set():
            with g.cv:
                while g.remaining > 0 and not stop.is_set() and (r in g.checked or g.outcome is not None):
                    g.cv.wait(poll)
                if g.remaining == 0 or stop.is_set():
                    return
                g.checked.add(r)
                if len(g.checked) == R:
                    g.outcome = resolve(g, s)
                    g.cv.notify_all()
                else:
                    while g.outcome is None and not stop.is_set():
                        g.cv.wait(poll)
                    if stop.is_set():
                        return
                kind, task, cost, ver = g.outcome
                g.acks += 1
                if g.acks == R:
                    g.checked.clear()
                    g.outcome = None
                    g.acks = 0
                    g.round += 1
                    g.cv.notify_all()
                else:
                    rid = g.round
                    while g.round == rid and not stop.is_set():
                        g.cv.wait(poll)
            if kind == "wait":
                with g.cv:
                    while g.version == ver and g.remaining > 0 and not stop.is_set():
                        g.cv.wait(poll)
                continue
            if cost:
                t0 = now_us()
                spin(cost * time_scale)
                if r == 0:
                    emit("coord", t0, now_us(), s, None, task if kind == "exec" else None)
            if kind == "defer":
                with g.cv:
                    while g.version == ver and g.remaining > 0 and not stop.is_set():
                        g.cv.wait(poll)
                continue
            t0 = now_us()
            spin((w["lat"][task] + inj.get(task, 0)) * time_scale)
            t1 = now_us()
            emit("exec", t0, t1, s, r if R > 1 else None, task)
            with g.cv:
                g.finishers += 1
                if g.finishers == R:
                    g.finishers = 0
                    g.sends = complete(g, s, task, t1)
                    g.finish_round += 1
                    g.cv.notify_all()
                else:
                    fr = g.finish_round
                    while g.finish_round == fr and not stop.is_set():
                        g.cv.wait(poll)
                sends = list(g.sends)
            for dtask, kind_e in sends:
                delay = comm_delay_sample(w["comm"], task, dtask, kind_e)
                if r == 0:
                    emit("send", t1, int(t1 + delay * time_scale), s, None, task)
                q = out_q[(s, r)]
                while not stop.is_set():
                    try:
                        q.put((dtask, delay), timeout=poll)
                        break
                    except queue.Full:
                        pass

    def sender(s, r):
        q = out_q[(s, r)]
        while not stop.is_set():
            try:
                dtask, delay = q.get(timeout=poll)
            except queue.Empty:
                continue
            if delay:
                time.sleep(delay * time_scale / 1e6)
            dq = in_q[(dtask[1], r)]
            while not stop.is_set():
                try:
                    dq.put(dtask, timeout=poll)
                    break
                except queue.Full:
                    pass

    def receiver(s, r):
        q = in_q[(s, r)]
        g = groups[s]
        while not stop.is_set():
            try:
                task = q.get(timeout=poll)
            except queue.Empty:
                continue
            if tp["skew_hi"] > 0 and R > 1:
                sk = int(substream(seed, "skew", task_key(task), r).integers(
                    tp["skew_lo"], tp["skew_hi"] + 1))
                if sk:
                    time.sleep(sk * time_scale / 1e6)
            t = now_us()
            mb, c = task[2], task[3]
            with g.cv:
                if task[0] == F:
                    g.views[r].fready.add((mb, c))
                elif (mb, c, F) in g.ctl.done:
                    g.views[r].bready.add((mb, c))
                else:
                    g.pend[r].add((mb, c))
                g.version += 1
                g.cv.notify_all()
            emit("recv", t, t, s, r, task)

    def watchdog():
        last, since = -1, time.monotonic()
        while not stop.is_set():
            time.sleep(0.05)
            if progress[0] != last:
                last, since = progress[0], time.monotonic()
            elif time.monotonic() - since > watchdog_secs:
                failure.append(f"watchdog: {progress[0]} tasks done")
                stop.set()
                return

    threads = []
    for s in range(n):
        for r in range(R):
            for fn, nm in ((worker, "compute"), (sender, "sender"), (receiver, "receiver")):
                threads.append(threading.Thread(target=fn, args=(s, r), daemon=True, name=nm))
    dog = threading.Thread(target=watchdog, daemon=True)
    for t in threads:
        t.start()
    dog.start()
    for t in threads:
        if t.name == "compute":
            t.join()
    stop.set()
    for t in threads:
        t.join(timeout=2.0)
    if failure:
        raise DeadlockError(failure[0])
    mk = max((e[1] for e in events if e[7] == "exec"), default=0)
    return events, mk


# ----------------------------------------------------------- validate -----
def validate(events, w, injected=None, slack=(0, 1.0, 0), clock="virtual", scale=1.0):
    """validate_trace, validate.py:44-132 -> list of (kind, detail) violations.

    ``events`` are 8-tuples (t0, t1, stage, rank, mb, chunk, dir, kind).
    """
    injected = injected or {}
    out = []
    sc = scale if clock == "wall" else 1.0
    lower, up_rel, up_abs = slack
    known = set()
    for s in range(w["N"]):
        for mb in range(w["M"]):
            for c in range(w["C"]):
                for d in ((F, B, W) if w["dec"] else (F, B)):
                    known.add((d, s, mb, c))
    by = {}
    cnt = {}
    ranks = set()
    for t0, t1, s, r, mb, c, d, kind in events:
        if kind != "exec":
            continue
        if t1 < t0:
            out.append(("malformed", f"exec ends before start at stage {s}"))
            continue
        t = (d, s, mb, c)
        if d is None or t not in known:
            out.append(("malformed", f"unknown task {t}"))
            continue
        rk = 0 if r is None else r
        ranks.add(rk)
        cnt[(t, rk)] = cnt.get((t, rk), 0) + 1
        by[(t, rk)] = (t0, t1, s)
    ranks = ranks or {0}
    for t in known:
        for rk in sorted(ranks):
            if cnt.get((t, rk), 0) != 1:
                out.append(("completeness", f"{task_key(t)} x{cnt.get((t, rk), 0)} rank {rk}"))
    for (t, rk), (t0, t1, s) in sorted(by.items()):
        exp = (w["lat"][t] + injected.get(t, 0)) * sc
        act = t1 - t0
        if act < exp - lower or act > exp * up_rel + up_abs:
            out.append(("duration", f"{task_key(t)} rank {rk}: {act} vs {exp}"))
    lanes = {}
    for (t, rk), (t0, t1, s) in by.items():
        lanes.setdefault((s, rk), []).append((t0, t1, t))
    for key, evs in sorted(lanes.items()):
        evs.sort()
        for a, b in zip(evs, evs[1:]):
            if b[0] < a[1]:
                out.append(("serialization", f"{key}: {task_key(a[2])} overlaps {task_key(b[2])}"))
    eps = 2 if clock == "wall" else 1e-9
    for src, dst, kind in task_graph(w):
        delay = comm_delay_sample(w["comm"], src, dst, kind) * sc
        for rk in sorted(ranks):
            a, b = by.get((src, rk)), by.get((dst, rk))
            if a is None or b is None:
                continue
            if b[0] < a[1] + delay - eps:
                out.append(("precedence", f"{kind} {task_key(src)}->{task_key(dst)} rank {rk}"))
    return out
