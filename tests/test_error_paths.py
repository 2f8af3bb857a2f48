"""Error paths of executeBatch (types.hpp:42-43): a livelock
budget that runs out raises LivelockError with the unfinished transactions
reported (ticket ~0) while the committed ones still replay bit-exactly; batch
sizes past the 30-bit priority range are refused before any input is read."""
import ctypes as C

import numpy as np
import pytest

from test_gpu_parity import check_replay, dev_factory  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def test_livelock_budget_reports_unfinished_transactions(hetm, orc, dev_factory):
    W, n = 64, 1 << 14  # every transaction fights over 64 accounts
    d = dev_factory(W, rs_gran_bytes=8, max_attempts=2)
    d.register_kernel(hetm.KERNEL_BANK)
    d.set_schedule(hetm.SCHED_OPTIMISTIC)  # SCAN never retries, so it cannot livelock
    init = np.full(W, 10_000, np.uint64)
    d.upload(hetm.REPLICA_DEV, 0, init)
    txs = orc.gen_bank_batch(7, n, 0, W)
    tickets = np.empty(n, np.uint64)
    st = hetm._lib.BatchStats()
    rc = hetm._lib.lib.hetm_dev_execute_batch_ex(d.h, hetm.KERNEL_BANK, txs.ctypes.data, 24, n, tickets.ctypes.data,
                                                 None, 0, C.byref(st))
    assert rc == hetm.LivelockError.code
    unfinished = tickets == np.uint64(2**64 - 1)
    assert st.livelocked == int(unfinished.sum()) > 0 and st.committed + st.livelocked == n
    # the committed subset is still a serializable batch: replay it in ticket order
    done = np.nonzero(~unfinished)[0]
    ref = init.copy()
    orc.bank_replay(ref, txs, done[np.argsort(tickets[done], kind="stable")], 8, 16384)
    assert (d.download(hetm.REPLICA_DEV) == ref).all()


def test_batch_past_the_priority_range_is_refused(hetm, dev_factory):
    d = dev_factory(64, rs_gran_bytes=8)
    d.register_kernel(hetm.KERNEL_BANK)
    one = np.zeros(1, hetm.BANK_TX)
    st = hetm._lib.BatchStats()
    rc = hetm._lib.lib.hetm_dev_execute_batch_ex(d.h, hetm.KERNEL_BANK, one.ctypes.data, 24, 1 << 30, None, None, 0,
                                                 C.byref(st))
    assert rc == hetm.InvalidSizeError.code
    rc = hetm._lib.lib.hetm_dev_execute_batch_dptr_ex(d.h, hetm.KERNEL_BANK, C.c_void_p(16), 1 << 30, C.c_void_p(16),
                                                      None, None)
    assert rc == hetm.InvalidSizeError.code
