"""One stage per PROCESS (torchrun, CUDA IPC mailboxes + peer flags) on the B200.

On a 1-GPU box both ranks share cuda:0 (RRFP_SAME_DEVICE=1): the IPC handle
exchange, the cross-process mailbox writes and flag releases are the same code
that runs one stage per GPU; only the link is local."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("hint", ["bf", "bfw"])
def test_two_process_pipeline_matches_single_process(hint):
    env = dict(os.environ, RRFP_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tools", "dist_check.py"), hint]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and line, p.stdout[-2000:] + p.stderr[-3000:]
    res = json.loads(line[-1])
    last = [r for r in res["ranks"] if r["rank"] == 1][0]
    ref = res["single_process_pp1_loss"]
    for l in last["losses"]:
        assert abs(l - ref) / ref < 1e-2, (l, ref)
    per_stage = 4 * (3 if hint == "bfw" else 2)
    assert all(r["n_exec"] == per_stage for r in res["ranks"])
