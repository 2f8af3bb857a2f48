"""Per-phase cycle breakdown of the bank batch kernel (run with HETM_KNOCKOUT=128 on the
experiments build: make -C paper_1905_00661_b200/csrc clean all EXPERIMENTS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_00661_b200 as hetm

W, B = 1 << 27, 1 << 20
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
for rep in range(3):
    txs = hetm.gen_bank_batch(10 + rep, B, 0, W // 2)
    r = d.execute_batch(hetm.KERNEL_BANK, txs, want_tickets=False)
    d.clear_round()
out = np.zeros(6, np.uint64)
hetm.check(hetm._lib.lib.hetm_dev_debug_words(d.h, out.ctypes.data, 6))
att = int(out[5])
print(f"kernel {r.kernel_ms:.3f} ms, aborts {r.aborts}, thread attempts {att}")
for i, name in enumerate(["P1 snapshot", "P2 prelock", "P3 ticket", "P4 validate+final", "P5 writeback"]):
    print(f"  {name:18s} {int(out[i]) / max(att, 1):9.0f} cycles / thread-attempt")
