"""The reference's own unit tests, run UNMODIFIED against this package.

A shim package named ``rrfp`` (written to a temp dir) re-exports this
package's modules under the reference's module names; the reference's test
files are copied next to it byte-for-byte and run with pytest in a
subprocess.  Covered: pkg/tests/test_arbitration.py (the ready-set arbiter
surface: StageBuffers / BackpressureState / StageProgress / ArbiterState /
next_by_priority / update_backpressure / arbitrate / advance_round_phase /
tp_coordinate, backed by the C twin), test_workload.py (task model,
generator) and test_jitter.py (injection tables; its paired-injection test
runs the replay engine through the host twin).

The reference tree exists only in the build container, so the test skips
elsewhere (the GPU box never sees /root/reference).
"""
import os
import shutil
import subprocess
import sys
import textwrap

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

SHIM = {
    "__init__.py": "from paper_2605_18750_b200 import *  # noqa\n",
    "arbitration.py": "from paper_2605_18750_b200.arbitration import *  # noqa\n",
    "workload.py": textwrap.dedent("""\
        from paper_2605_18750_b200.workload import *  # noqa
        from paper_2605_18750_b200.workload import (BACKWARD, FORWARD, WEIGHT, CommDelay,  # noqa
            DependencyEdge, DistSpec, GeneratorSpec, TaskId, Workload, WorkloadError,
            build_task_graph, constant, generate_workload, lognormal, topological_order, uniform)
        """),
    "jitter.py": "from paper_2605_18750_b200.jitter import *  # noqa\n"
                 "from paper_2605_18750_b200.jitter import (PRESETS, JitterConfig, JitterState,  # noqa\n"
                 "    build_injection_table, ema_update, sample_delay)\n",
    "rng.py": "from paper_2605_18750_b200.rng import substream  # noqa\n",
    # CPU-only container: the virtual-clock engine runs on the host twin of the
    # device state machine (an explicit device choice, never a silent fallback)
    "engine.py": textwrap.dedent("""\
        from paper_2605_18750_b200 import engine as _e
        from paper_2605_18750_b200.engine import EngineDeadlockError  # noqa

        def run_rrfp(*a, **k):
            k.setdefault("device", "cpu")
            return _e.run_rrfp(*a, **k)
        """),
    "baselines.py": textwrap.dedent("""\
        from paper_2605_18750_b200 import engine as _e
        from paper_2605_18750_b200.baselines import *  # noqa
        from paper_2605_18750_b200.baselines import (FixedSchedule, ScheduleDeadlockError,  # noqa
            build_1f1b_schedule)

        def run_fixed(*a, **k):
            k.setdefault("device", "cpu")
            return _e.run_fixed(*a, **k)
        """),
}

FILES = ["test_workload.py", "test_arbitration.py", "test_jitter.py"]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not mounted (GPU box)")
def test_reference_unit_tests_pass_unmodified(tmp_path):
    pkg = tmp_path / "rrfp"
    pkg.mkdir()
    for name, body in SHIM.items():
        (pkg / name).write_text(body)
    for f in FILES:
        shutil.copyfile(os.path.join(REF_TESTS, f), tmp_path / f)   # byte-identical copies
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path), ROOT]))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *FILES],
                       cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    assert " passed" in p.stdout and "failed" not in p.stdout
