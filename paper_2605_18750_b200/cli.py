"""Command line for the B200 path: the reference's run commands with a ``--gpu`` hook.

    python -m paper_2605_18750_b200 simulate-rrfp [--config] CONFIG [--gpu] [--live] [--set a.b=v ...]
    python -m paper_2605_18750_b200 simulate-1f1b [--config] CONFIG [--gpu]
    python -m paper_2605_18750_b200 live          [--config] CONFIG

Mirrors ``rrfp.cli`` (cli.py:106-273) for these three commands: the same
config resolution and flags (--seed --hint --limit --jitter --tp --out
--watchdog-secs --set), artifacts under ``<out>/<run-id>/`` (config.json,
trace.jsonl, metrics.json, reports/gantt.csv), a one-line summary, and the
exit codes 0 ok / 2 config violation (incl. a missing or malformed config
file) / 3 deadlock or watchdog with ``<out>/deadlock_dump.txt`` (cli.py:37-39,
326-338).
``simulate-*`` run the virtual clock on the host twin of the C++ state
machine, or with ``--gpu`` in the device replay kernel; ``live`` runs the
device lanes (gpu.mode free|fixed|replay).  Unlike the reference
 an interleaved / decomposed 1F1B request exits 2.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

from .baselines import ScheduleDeadlockError, build_1f1b_schedule
from .config import ConfigError, RunConfig, apply_overrides, resolve_config
from .engine import EngineDeadlockError, run_fixed, run_rrfp
from .jitter import build_injection_table

EXIT_OK, EXIT_CONFIG, EXIT_DEADLOCK = 0, 2, 3

DEFAULT_DOC = {"generator": {"num_stages": 4, "num_microbatches": 8,
                             "forward": {"kind": "uniform", "lo": 80, "hi": 120},
                             "backward": {"kind": "uniform", "lo": 80, "hi": 120}}}


def _resolve(args) -> RunConfig:
    doc = DEFAULT_DOC
    if args.config:
        with open(args.config) as f:
            doc = json.load(f)
    sets = list(args.set or [])
    flag_paths = (("seed", "seed"), ("hint", "scheduler.hint"), ("limit", "scheduler.buffer_limit"),
                  ("out", "output.dir"), ("watchdog_secs", "live.watchdog_secs"))
    for attr, path in flag_paths:
        v = getattr(args, attr, None)
        if v is not None:
            sets.append(f"{path}={v}")
    if args.jitter is not None:
        if args.jitter.startswith("file:"):
            sets.append(f"jitter={Path(args.jitter[5:]).read_text().strip()}")
        else:
            sets.append(f"jitter={args.jitter}")
    if args.tp is not None:
        sets.append(("workload" if "workload" in doc else "generator") + f".tp_group_size={args.tp}")
    return resolve_config(apply_overrides(doc, sets))


def write_gantt(trace, path) -> None:
    """One row per executed task: stage, rank, microbatch, chunk, direction, t_start, t_end."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["stage", "rank", "microbatch", "chunk", "direction", "t_start", "t_end"])
        for e in trace.events:
            if e.event_kind == "exec":
                w.writerow([e.stage, "" if e.rank is None else e.rank, e.microbatch, e.chunk,
                            e.direction, e.t_start, e.t_end])


def write_run(cfg: RunConfig, trace, metrics, extra: dict | None = None) -> Path:
    d = Path(cfg.output_dir) / cfg.run_id()
    (d / "reports").mkdir(parents=True, exist_ok=True)
    (d / "config.json").write_text(json.dumps(cfg.raw, indent=2, sort_keys=True))
    trace.dump_jsonl(d / "trace.jsonl")
    metrics.dump(d / "metrics.json")
    write_gantt(trace, d / "reports" / "gantt.csv")
    if extra:
        (d / "reports" / "summary.json").write_text(json.dumps(extra, indent=2, sort_keys=True))
    return d


def _simulate(cfg: RunConfig, kind: str, device: str):
    if kind == "1f1b":
        w = cfg.workload
        if w.num_chunks > 1 or w.decompose_backward:
            raise ConfigError("scheduler.kind", "1f1b needs num_chunks == 1 and no decomposed backward")
        inj = build_injection_table(w, cfg.jitter, cfg.seed)
        return run_fixed(build_1f1b_schedule(w), w, injected_delays=inj, device=device)
    return run_rrfp(cfg.workload, cfg.hint, cfg.buffer_limit, cfg.seed, jitter=cfg.jitter, tp=cfg.tp,
                    device=device)


def _summary(cmd, cfg, metrics, d):
    return (f"{cmd} run={cfg.run_id()} makespan={metrics.makespan} "
            f"bubble={metrics.bubble_fraction():.4f} out={d}")


def cmd_simulate(args, kind: str) -> int:
    args.set = list(args.set or []) + [f"scheduler.kind={kind}"]
    if kind == "rrfp" and getattr(args, "live", False):     # cli.py:187-188
        return cmd_live(args)
    cfg = _resolve(args)
    trace, metrics = _simulate(cfg, kind, "cuda" if args.gpu else "cpu")
    d = write_run(cfg, trace, metrics, {"device": "cuda" if args.gpu else "cpu (host twin)"})
    print(_summary(f"simulate-{kind}", cfg, metrics, d))
    return EXIT_OK


def cmd_live(args) -> int:
    from .runtime import run_gpu
    cfg = _resolve(args)
    sched = build_1f1b_schedule(cfg.workload) if cfg.gpu_mode == "fixed" else None
    dev = cfg.gpu_device
    placement = [[dev] * cfg.workload.tp_group_size for _ in range(cfg.workload.num_stages)]
    trace, metrics = run_gpu(cfg.workload, cfg.hint, cfg.buffer_limit, cfg.time_scale, seed=cfg.seed,
                             jitter=cfg.jitter, tp=cfg.tp, watchdog_secs=cfg.watchdog_secs,
                             mode=cfg.gpu_mode, schedule=sched, placement=placement)
    d = write_run(cfg, trace, metrics, {"device": f"cuda:{dev}", "mode": cfg.gpu_mode})
    print(_summary("live", cfg, metrics, d))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2605_18750_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("simulate-rrfp", "simulate-1f1b", "live"):
        p = sub.add_parser(name)
        p.add_argument("config", nargs="?")
        p.add_argument("--config", dest="config_opt", metavar="CONFIG",
                       help="JSON config path (the reference's spelling, cli.py:277)")
        p.add_argument("--live", action="store_true",
                       help="simulate-rrfp: execute on the device lanes instead (cli.py:187-188)")
        p.add_argument("--set", action="append", metavar="KEY.PATH=VALUE")
        p.add_argument("--seed", type=int)
        p.add_argument("--hint")
        p.add_argument("--limit", type=int)
        p.add_argument("--jitter")
        p.add_argument("--tp", type=int)
        p.add_argument("--out")
        p.add_argument("--watchdog-secs", dest="watchdog_secs", type=float)
        p.add_argument("--gpu", action="store_true",
                       help="simulate on the device replay kernel (live always runs on the device)")
    return ap


def _write_dump(args, e) -> Path:
    """The reference's deadlock artefact (cli.py:332-338): <out>/deadlock_dump.txt."""
    path = Path(getattr(args, "out", None) or "out") / "deadlock_dump.txt"
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(str(getattr(e, "dump", "") or e) + "\n")
    return path


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.config_opt is not None:
        if args.config is not None and args.config != args.config_opt:
            print("config error: give the config once (positional or --config)", file=sys.stderr)
            return EXIT_CONFIG
        args.config = args.config_opt
    try:
        if args.cmd == "live":
            return cmd_live(args)
        return cmd_simulate(args, "rrfp" if args.cmd == "simulate-rrfp" else "1f1b")
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except (json.JSONDecodeError, FileNotFoundError) as e:   # cli.py:329-331
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except (EngineDeadlockError, ScheduleDeadlockError) as e:
        print(f"deadlock/watchdog: {e} (dump: {_write_dump(args, e)})", file=sys.stderr)
        return EXIT_DEADLOCK
    except Exception as e:   # the runtime's watchdog (LiveWatchdogError) -> exit 3 with its dump
        if type(e).__name__ == "LiveWatchdogError":
            print(f"deadlock/watchdog: {e} (dump: {_write_dump(args, e)})", file=sys.stderr)
            return EXIT_DEADLOCK
        raise


if __name__ == "__main__":
    sys.exit(main())
