"""Config schema (rrfp.config) and the CLI --gpu hook (rrfp.cli), host-side.

Golden run ids / makespans come from the reference run here (SURVEY App. B:
CLI on configs/example.json -> rrfp 2158 us, 1f1b 2289 us); the bundled
configs are restated inline (the GPU box has no /root/reference)."""
import json

import pytest

import paper_2605_18750_b200 as P
from paper_2605_18750_b200.cli import main

EXAMPLE = {"seed": 1, "generator": {"num_stages": 4, "num_microbatches": 8,
                                    "forward": {"kind": "uniform", "lo": 80, "hi": 120},
                                    "backward": {"kind": "uniform", "lo": 80, "hi": 120}},
           "scheduler": {"kind": "rrfp", "hint": "bf", "buffer_limit": 32}, "jitter": "J0",
           "output": {"dir": "out"}}
INTERLEAVED_TP = {"seed": 7, "generator": {"num_stages": 4, "num_microbatches": 8, "num_chunks": 2,
                                           "tp_group_size": 2,
                                           "forward": {"kind": "lognormal", "mu": 4.8, "sigma": 0.4, "lo": 40, "hi": 400},
                                           "backward": {"kind": "lognormal", "mu": 5.0, "sigma": 0.4, "lo": 40, "hi": 500},
                                           "comm_delay": {"kind": "uniform", "lo": 5, "hi": 30, "seed": 7}},
                  "scheduler": {"kind": "rrfp", "hint": "bf", "buffer_limit": 8},
                  "tp": {"coordination_round_cost": 5, "skew_lo": 0, "skew_hi": 20}, "jitter": "J1",
                  "output": {"dir": "out"}}
HEAVY_MM = {"seed": 3, "generator": {"num_stages": 8, "num_microbatches": 24,
                                     "forward": {"kind": "uniform", "lo": 150, "hi": 250},
                                     "backward": {"kind": "uniform", "lo": 150, "hi": 250}, "heavy_prefix": 2.5},
            "scheduler": {"kind": "rrfp", "hint": "bf", "buffer_limit": 32}, "output": {"dir": "out"}}


@pytest.mark.parametrize("doc,run_id", [(EXAMPLE, "47c91a024b90"), (INTERLEAVED_TP, "daf3d8c0e519"),
                                        (HEAVY_MM, "2c23af862eac")])
def test_run_ids_match_reference(doc, run_id):
    assert P.resolve_config(doc).run_id() == run_id


def test_resolved_fields():
    cfg = P.resolve_config(INTERLEAVED_TP)
    assert cfg.workload.num_chunks == 2 and cfg.workload.tp_group_size == 2
    assert cfg.buffer_limit == 8 and cfg.tp.skew_hi == 20 and cfg.jitter == P.JITTER_PRESETS["J1"]
    assert cfg.gpu_mode == "free" and cfg.gpu_device == 0
    gcfg = P.resolve_config({**EXAMPLE, "gpu": {"mode": "replay"}})
    assert gcfg.gpu_mode == "replay" and gcfg.run_id() != P.resolve_config(EXAMPLE).run_id()


@pytest.mark.parametrize("doc,path", [
    ({"seed": 0}, "workload"),
    ({**EXAMPLE, "workload": {}}, "workload"),
    ({**EXAMPLE, "seed": True}, "seed"),
    ({**EXAMPLE, "scheduler": {"hint": "zz"}}, "scheduler.hint"),
    ({**EXAMPLE, "scheduler": {"kind": "gpipe"}}, "scheduler.kind"),
    ({**EXAMPLE, "scheduler": {"buffer_limit": 0}}, "scheduler.buffer_limit"),
    ({**EXAMPLE, "jitter": "J9"}, "jitter"),
    ({**EXAMPLE, "live": {"time_scale": 0}}, "live.time_scale"),
    ({**EXAMPLE, "gpu": {"mode": "warp"}}, "gpu.mode"),
])
def test_config_errors_name_the_field(doc, path):
    with pytest.raises(P.ConfigError) as e:
        P.resolve_config(doc)
    assert e.value.path == path


def test_overrides():
    doc = P.apply_overrides(EXAMPLE, ["scheduler.hint=fb", "seed=5", "live.watchdog_secs=2.5"])
    cfg = P.resolve_config(doc)
    assert cfg.hint.kind == "fb" and cfg.seed == 5 and cfg.watchdog_secs == 2.5
    with pytest.raises(P.ConfigError):
        P.apply_overrides(EXAMPLE, ["nonsense"])


@pytest.mark.parametrize("cmd,makespan", [("simulate-rrfp", 2158), ("simulate-1f1b", 2289)])
def test_cli_simulate_host_twin(tmp_path, capsys, cmd, makespan):
    cfgp = tmp_path / "example.json"
    cfgp.write_text(json.dumps(EXAMPLE))
    rc = main([cmd, str(cfgp), "--out", str(tmp_path / "out")])
    assert rc == 0
    line = capsys.readouterr().out.strip()
    assert f"makespan={makespan}" in line
    run = next((tmp_path / "out").iterdir())
    assert {p.name for p in run.iterdir()} >= {"config.json", "trace.jsonl", "metrics.json", "reports"}
    gantt = (run / "reports" / "gantt.csv").read_text().splitlines()
    assert gantt[0].startswith("stage,rank,microbatch") and len(gantt) == 1 + 4 * 8 * 2
    assert json.loads((run / "metrics.json").read_text())["makespan"] == makespan


def test_cli_exit_codes(tmp_path, capsys):
    cfgp = tmp_path / "il.json"
    cfgp.write_text(json.dumps(INTERLEAVED_TP))
    # the reference crashes here with a traceback; the contract says exit 2
    assert main(["simulate-1f1b", str(cfgp), "--out", str(tmp_path)]) == 2
    assert main(["simulate-rrfp", str(cfgp), "--set", "scheduler.buffer_limit=0", "--out", str(tmp_path)]) == 2
    ext = tmp_path / "hint.json"
    ext.write_text(json.dumps({"order": [["F", "asc"]]}))     # never schedules B: deadlock
    assert main(["simulate-rrfp", "--hint", f"file:{ext}", "--out", str(tmp_path)]) == 3


def test_cli_reference_spelling_and_errors(tmp_path, capsys):
    """`--config PATH` (the reference's documented form, cli.py:277) works; a
    missing or malformed config exits 2 (cli.py:329-331); a deadlock exits 3
    and writes <out>/deadlock_dump.txt (cli.py:332-338)."""
    cfgp = tmp_path / "example.json"
    cfgp.write_text(json.dumps(EXAMPLE))
    assert main(["simulate-rrfp", "--config", str(cfgp), "--out", str(tmp_path / "o")]) == 0
    assert "makespan=2158" in capsys.readouterr().out
    assert main(["simulate-rrfp", "--config", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert main(["simulate-1f1b", "--config", str(bad)]) == 2
    ext = tmp_path / "hint.json"
    ext.write_text(json.dumps({"order": [["F", "asc"]]}))
    out = tmp_path / "dl"
    assert main(["simulate-rrfp", "--hint", f"file:{ext}", "--out", str(out)]) == 3
    dump = (out / "deadlock_dump.txt").read_text()
    assert "remaining" in dump


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["free", "fixed", "replay"])
def test_cli_gpu_hook(tmp_path, capsys, mode):
    """--gpu: the replay kernel gives the host twin's makespan; live runs the device lanes."""
    cfgp = tmp_path / "example.json"
    cfgp.write_text(json.dumps({**EXAMPLE, "gpu": {"mode": mode, "device": 0}}))
    assert main(["simulate-rrfp", str(cfgp), "--gpu", "--out", str(tmp_path / "sim")]) == 0
    assert "makespan=2158" in capsys.readouterr().out
    assert main(["live", str(cfgp), "--out", str(tmp_path / "live")]) == 0
    run = next((tmp_path / "live").iterdir())
    rows = (run / "reports" / "gantt.csv").read_text().splitlines()
    assert len(rows) == 1 + 4 * 8 * 2
