"""Bank kernel under heavy lock-stripe false sharing (phased_tx.cuh KO_STRIPES):
a 1024-stripe table over 2^16 words (64 words per stripe, HETM_STRIPE_BITS=10,
read once per process, hence a subprocess) makes most transactions meet a
stripe held or versioned by an unrelated transfer.  The batch must still
commit every transaction (priority rule), replay bit-exactly in ticket order
on the oracle (STMR, RS/WS/ChunkMap), and keep the bank sum."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1905_00661_b200 as hetm
import oracle as orc
out = []
for W, n, gran, seed in ((1 << 16, 1 << 14, 8, 3), (1 << 16, 1 << 15, 1024, 4), (1 << 18, 1 << 16, 64, 5)):
    with hetm.GpuDevice(W, rs_gran_bytes=gran) as d:
        d.register_kernel(hetm.KERNEL_BANK)
        d.set_schedule(hetm.SCHED_OPTIMISTIC)
        init = np.full(W, 1000, np.uint64)
        d.upload(hetm.REPLICA_DEV, 0, init)
        txs = orc.gen_bank_batch(seed, n, 0, W)
        r = d.execute_batch(hetm.KERNEL_BANK, txs)
        order = orc.order_by_ticket(r.tickets)
        ref = init.copy()
        rs, ws, ch = orc.bank_replay(ref, txs, order, gran, 16384)
        got = d.download(hetm.REPLICA_DEV)
        out.append({"W": W, "n": n, "committed": int(r.committed), "aborts": int(r.aborts),
                    "unique_tickets": int(len(np.unique(r.tickets))), "replay": bool((got == ref).all()),
                    "rs": bool((d.snapshot(hetm.BMP_RS).words == rs).all()),
                    "ws": bool((d.snapshot(hetm.BMP_WS).words == ws).all()),
                    "chunk": bool((d.snapshot(hetm.BMP_CHUNK).words == ch).all()),
                    "sum": bool(int(got.sum(dtype=np.uint64)) == 1000 * W)})
print(json.dumps(out))
"""


@pytest.mark.gpu
def test_bank_batch_under_heavy_stripe_sharing():
    env = dict(os.environ, HETM_STRIPE_BITS="10")
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr
    for case in json.loads(p.stdout.strip().splitlines()[-1]):
        assert case["committed"] == case["n"] == case["unique_tickets"], case
        assert case["aborts"] > 0, case  # the sharing is real
        assert case["replay"] and case["rs"] and case["ws"] and case["chunk"] and case["sum"], case
