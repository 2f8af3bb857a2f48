"""Device submission queue + GPU-controller launch rule (
include/hetm_b200/dispatch.hpp): the CPU unit test of the rule, and live
engine rounds fed from the queue (GPU), replayed bit-exactly on the oracle."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _exe(name):
    p = os.path.join(ROOT, "build", name)
    if not os.path.exists(p):
        pytest.skip(f"build/{name} not built (run __graft_entry__.build())")
    return p


def test_queue_launch_rule_cpu():
    """batchSize-1 -> no batch, batchSize -> exactly batchSize (FIFO); 8 producers x 10^4
    requests consumed exactly once; the max-wait knob releases a partial batch."""
    out = subprocess.run([_exe("dispatch_test")], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr


@pytest.mark.gpu
def test_queue_fed_rounds():
    out = subprocess.run([_exe("queue_round_test"), "5", "4096"], capture_output=True, text=True, timeout=600)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout + out.stderr
    r = json.loads(lines[-1])
    assert r["ok"] == 1 and r["batches"] >= 5 and r["executed"] + r["queued_tail"] == r["submitted"]
